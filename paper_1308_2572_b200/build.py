"""Build libara.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_1308_2572_b200.build      # or __graft_entry__.build()

Writes ``paper_1308_2572_b200/libara.so`` and ``build/ptxas_*.txt`` (register / spill report of
every kernel, kept for review).  Re-compiles only when a source or header is newer than the
library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libara.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-fno-fast-math",
          "-I", INCLUDE, "-I", CSRC]
# -fmad=false: no FMA contraction anywhere (the kernels also use __dmul_rn/__dsub_rn/__dadd_rn
# explicitly); the oracle's reading R7 fixes separately rounded products and differences.
PER_FILE = {
    "scan.cu": ["-fmad=false", "-Xptxas", "-v"],
    "scan_pair.cu": ["-fmad=false", "-Xptxas", "-v"],
    "portfolio.cu": ["-fmad=false", "-Xptxas", "-v"],
    "hoist.cu": ["-fmad=false", "-Xptxas", "-v"],
    "metrics.cu": ["-Xptxas", "-v"],
    "ara.cpp": [],
}


def _sources():
    return [os.path.join(CSRC, f) for f in PER_FILE]


def source_sha16() -> str:
    """Hash of everything that determines libara.so's machine code: the kernel and host sources,
    the internal headers, the public header and this script (flags).  nvcc output is not
    byte-reproducible, so committed ncu counters are keyed by this instead of the binary."""
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(CSRC, "*")) + [os.path.join(INCLUDE, "ara.h"),
                                                          os.path.abspath(__file__)])
    for f in files:
        if os.path.isfile(f) and not f.endswith((".o", ".so")):
            h.update(os.path.basename(f).encode())
            with open(f, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = _sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(
        os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "ara.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "",
          defines: tuple = (), extra: tuple = ()) -> str:
    """Build libara.so; ``variant`` + ``defines`` (+ ``extra`` nvcc flags for the kernel files)
    build a tuning library libara_<variant>.so (loaded by the binding when
    ARA_LIB_VARIANT=<variant>)."""
    lib = LIB if not variant else os.path.join(PKG, f"libara_{variant}.so")
    if not variant and not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs, procs = [], []
    for src in _sources():  # the translation units compile in parallel
        name = os.path.basename(src)
        obj = os.path.join(BUILD, (f"{variant}_" if variant else "") + name + ".o")
        cmd = [NVCC, *ARCH, *COMMON, *[f"-D{d}" for d in defines], *PER_FILE[name], *extra,
               "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, *COMMON, *[f"-D{d}" for d in defines], "-x", "cu", *ARCH, "-c", src,
                   "-o", obj]
        procs.append((name, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                  stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    failed = None
    for name, cmd, pr in procs:
        out, err = pr.communicate()
        with open(os.path.join(BUILD, f"ptxas_{variant}{name}.txt"), "w") as f:
            f.write(" ".join(cmd) + "\n" + out + err)
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            failed = failed or name
        elif verbose:
            sys.stdout.write(err)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_1308_2572_b200.build [--force] [-v] [--variant NAME -DFOO=1 ...
    #                                      --nvcc=-maxrregcount=144 ...]
    a = sys.argv[1:]
    var = a[a.index("--variant") + 1] if "--variant" in a else ""
    print(build(force="--force" in a, verbose="-v" in a, variant=var,
                defines=tuple(x[2:] for x in a if x.startswith("-D")),
                extra=tuple(x[7:] for x in a if x.startswith("--nvcc="))))
