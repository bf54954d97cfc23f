"""C-ABI library: builds, loads and exports every symbol include/ara.h declares (no GPU needed);
host-side argument validation paths that do not touch the device."""
import ctypes
import os
import re

import pytest

from paper_1308_2572_b200 import ara, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ara.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ara_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    path = build.build()
    assert os.path.exists(path)
    lib = ctypes.CDLL(path)
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), f"libara.so does not export {name}"
    assert sorted(ara.EXPORTS) == decl  # the binding covers the whole ABI


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB],
                          capture_output=True, text=True).stdout
    assert "LDG.E.ENL2.256" in sass or "ENL2.256" in sass  # 256-bit row gathers (sm_100+)
    assert "DFMA" not in sass.split("metrics_kernel")[0]   # no contraction in the scan


def test_status_strings_and_null_handling():
    L = ara.lib()
    for code, name in ara.STATUS_NAMES.items():
        assert ara.ara_status_string(code) == name
    assert L.ara_load_elts(None, 10, 1, None, None, None, None) == 1  # ARA_ERR_ARG
    assert L.ara_run(None, 1, None, None, None, 0, 0) == 1
    assert L.ara_metrics(None, None, 0, 0, None, None, None) == 1
    L.ara_destroy(None)
    assert L.ara_last_error(None) == b"NULL context"
    out = ctypes.c_void_p()
    assert L.ara_create(0, None, None) == 1


def test_no_gpu_fails_loudly_not_silently():
    """Without a GPU ara_create must fail (there is no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ara.AraError) as ei:
        ara.Context(0)
    assert ei.value.status_name in ("ARA_ERR_CUDA",)


def test_binding_refuses_missing_library(monkeypatch, tmp_path):
    monkeypatch.setattr(ara, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(ara, "_lib", None)
    with pytest.raises(ara.AraLibraryMissing):
        ara.lib()


@pytest.mark.parametrize("cname,pyname", [("ara_fin_terms", "FinTerms"),
                                          ("ara_layer_terms", "LayerTerms"),
                                          ("ara_outputs", "Outputs"), ("ara_info", "Info")])
def test_binding_structs_match_header_layout(tmp_path, cname, pyname):
    """Every struct the binding passes across the ABI has the header's size and field offsets
    (compiled with the host C compiler from include/ara.h)."""
    import subprocess
    st = getattr(ara, pyname)
    fields = [f for f, _ in st._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stddef.h>\n#include <stdio.h>\n#include \"ara.h\"\nint main(void){\n"
                   f"  printf(\"%zu\\n\", sizeof({cname}));\n"
                   + "".join(f"  printf(\"%zu\\n\", offsetof({cname}, {f}));\n" for f in fields)
                   + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src),
                           "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)], text=True).split()]
    assert got[0] == ctypes.sizeof(st)
    assert got[1:] == [getattr(st, f).offset for f in fields]


def _build_c_example(tmp_path):
    import subprocess
    exe = tmp_path / "ara_example"
    pkg = os.path.join(ROOT, "paper_1308_2572_b200")
    build.build()
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I",
                           os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "ara_example.c"), "-L", pkg, "-lara",
                           f"-Wl,-rpath,{pkg}", "-o", str(exe)])
    return exe


def test_c_example_links_and_fails_loudly_without_gpu(tmp_path):
    """examples/ara_example.c compiles against include/ara.h alone and links libara.so; without a
    GPU ara_create reports ARA_ERR_CUDA (no CPU fallback)."""
    import subprocess
    import torch
    exe = _build_c_example(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("GPU present: see test_c_example_on_gpu")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "ARA_ERR_CUDA" in r.stderr


@pytest.mark.gpu
def test_c_example_on_gpu(tmp_path):
    """The C example on the GPU prints SPEC.md's worked-example YLT [[150, 0]] (L252-L262)."""
    import subprocess
    exe = _build_c_example(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "YLT 150 0" in r.stdout
