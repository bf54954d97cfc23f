"""Thin Python binding of ``include/ara.h`` (argument marshalling only).

Every function has the C name and forwards to ``libara.so``; every step of the method runs in the
library's CUDA kernels.  Device arrays are torch CUDA tensors (PyTorch supplies device memory and
streams only); host arrays are numpy arrays or CPU tensors.  There is no CPU fallback: if the
library is not built, importing this module raises ``AraLibraryMissing``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libara.so")

ARA_OK = 0
STATUS_NAMES = {0: "ARA_OK", 1: "ARA_ERR_ARG", 2: "ARA_ERR_RANGE", 3: "ARA_ERR_VALIDATION",
                4: "ARA_ERR_STATE", 5: "ARA_ERR_EMPTY", 6: "ARA_ERR_OOM", 7: "ARA_ERR_CUDA",
                8: "ARA_ERR_UNSUPPORTED"}
ARA_RUN_SYNC = 1
ARA_RUN_VALIDATE = 2
ARA_RUN_BALANCE = 4
ARA_RUN_HOIST = 8
ARA_MAX_ELTS_PER_LAYER = 64
ARA_MAX_P = 32

# Every symbol include/ara.h declares (tests check the library exports all of them).
EXPORTS = ["ara_status_string", "ara_create", "ara_set_precision", "ara_set_stream", "ara_destroy", "ara_last_error",
           "ara_load_elts", "ara_set_layers", "ara_run", "ara_run_outputs", "ara_run_host",
           "ara_synchronize",
           "ara_metrics", "ara_metrics_host", "ara_metrics_rows", "ara_metrics_sharded",
           "ara_portfolio_ylt", "ara_ep_curve",
           "ara_get_info",
           "ara_layer_store_shape",
           "ara_export_store"]


# int reduce(uint64_t offset, uint64_t count, int is_f64, void *user)   (include/ara.h)
SHARD_REDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                ctypes.c_void_p)


class AraLibraryMissing(ImportError):
    pass


class AraError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        self.status_name = STATUS_NAMES.get(status, str(status))
        super().__init__(f"{self.status_name}: {message}")


class FinTerms(ctypes.Structure):
    _fields_ = [("rate", ctypes.c_double), ("retention", ctypes.c_double),
                ("limit", ctypes.c_double)]


class LayerTerms(ctypes.Structure):
    _fields_ = [("occ_retention", ctypes.c_double), ("occ_limit", ctypes.c_double),
                ("agg_retention", ctypes.c_double), ("agg_limit", ctypes.c_double)]


class Outputs(ctypes.Structure):
    _fields_ = [("ylt", ctypes.c_void_p), ("ylt_ld", ctypes.c_uint64),
                ("max_occ", ctypes.c_void_p), ("max_occ_ld", ctypes.c_uint64),
                ("event_inc", ctypes.c_void_p), ("event_inc_ld", ctypes.c_uint64)]


class Info(ctypes.Structure):
    _fields_ = [("catalogue_size", ctypes.c_uint32), ("n_elts", ctypes.c_uint32),
                ("n_layers", ctypes.c_uint32), ("max_row_width", ctypes.c_uint32),
                ("store_bytes", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("device", ctypes.c_int), ("sm_count", ctypes.c_int),
                ("row_addressing", ctypes.c_int), ("layer_kernel", ctypes.c_int),
                ("gather_row_bytes", ctypes.c_uint32), ("last_kernel", ctypes.c_char * 64)]


def _load() -> ctypes.CDLL:
    path = LIB_PATH
    variant = os.environ.get("ARA_LIB_VARIANT")  # tuning builds: libara_<variant>.so (build.py)
    if variant:
        path = os.path.join(_PKG, f"libara_{variant}.so")
    if not os.path.exists(path):
        raise AraLibraryMissing(
            f"{path} is not built; run `python -m paper_1308_2572_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    p, u32, u64, i32, d = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                           ctypes.c_double)
    sig = {
        "ara_status_string": ([i32], ctypes.c_char_p),
        "ara_create": ([i32, p, ctypes.POINTER(p)], i32),
        "ara_set_stream": ([p, p], i32),
        "ara_set_precision": ([p, u32], i32),
        "ara_destroy": ([p], None),
        "ara_last_error": ([p], ctypes.c_char_p),
        "ara_load_elts": ([p, u32, u32, p, p, p, p], i32),
        "ara_set_layers": ([p, u32, p, p, p], i32),
        "ara_run": ([p, u64, p, p, p, u64, u32], i32),
        "ara_run_outputs": ([p, u64, p, p, ctypes.POINTER(Outputs), u32], i32),
        "ara_run_host": ([p, u64, p, p, p, u64, u32], i32),
        "ara_synchronize": ([p], i32),
        "ara_metrics": ([p, p, u64, u32, p, p, p], i32),
        "ara_metrics_host": ([p, p, u64, u32, p, p, p], i32),
        "ara_portfolio_ylt": ([p, p, u64, u64, p, u32], i32),
        "ara_ep_curve": ([p, p, u64, p], i32),
        "ara_metrics_rows": ([p, p, u32, u64, u64, u32, p, p, p], i32),
        "ara_metrics_sharded": ([p, p, u64, u64, u32, p, p, p, p, u64, SHARD_REDUCE, p], i32),
        "ara_get_info": ([p, ctypes.POINTER(Info)], i32),
        "ara_layer_store_shape": ([p, u32, ctypes.POINTER(u32), ctypes.POINTER(u32)], i32),
        "ara_export_store": ([p, u32, p, p], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _host(a, dtype) -> np.ndarray:
    if hasattr(a, "is_cuda"):  # torch tensor
        if a.is_cuda:
            raise TypeError("expected a host array, got a CUDA tensor")
        a = a.numpy()
    return np.ascontiguousarray(a, dtype=dtype)


def _hptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _dptr(t, dtype_name: str):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if str(t.dtype) != dtype_name:
        raise TypeError(f"expected {dtype_name}, got {t.dtype}")
    if not t.is_contiguous():
        raise TypeError("expected a contiguous tensor")
    return t.data_ptr() if t.numel() else None


class Context:
    """Owns one ``ara_ctx`` on a CUDA device / stream."""

    def __init__(self, device: int = 0, stream=None):
        self._ptr = ctypes.c_void_p()
        handle = None
        if stream is not None:
            handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        st = lib().ara_create(int(device), handle, ctypes.byref(self._ptr))
        if st != ARA_OK:
            raise AraError(st, "ara_create failed")
        self.device = device
        self.stream = stream

    def _check(self, st: int):
        if st != ARA_OK:
            raise AraError(st, lib().ara_last_error(self._ptr).decode())

    def close(self):
        if self._ptr:
            lib().ara_destroy(self._ptr)
            self._ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ calls
    def ara_set_precision(self, bits: int):
        self._check(lib().ara_set_precision(self._ptr, int(bits)))

    def ara_set_stream(self, stream):
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self._check(lib().ara_set_stream(self._ptr, handle))

    def ara_load_elts(self, catalogue_size: int, rec_offsets, rec_event_ids, rec_losses, fin):
        ro = _host(rec_offsets, np.uint64)
        ids = _host(rec_event_ids, np.uint32)
        ls = _host(rec_losses, np.float64)
        f = _host(fin, np.float64).reshape(-1, 3)
        self._check(lib().ara_load_elts(self._ptr, int(catalogue_size), ro.shape[0] - 1, _hptr(ro),
                                        _hptr(ids), _hptr(ls), _hptr(f)))

    def ara_set_layers(self, layer_terms, elt_offsets, elt_index):
        lt = _host(layer_terms, np.float64).reshape(-1, 4)
        eo = _host(elt_offsets, np.uint32)
        ei = _host(elt_index, np.uint32)
        self._check(lib().ara_set_layers(self._ptr, eo.shape[0] - 1, _hptr(lt), _hptr(eo),
                                         _hptr(ei)))

    def ara_run(self, d_trial_offsets, d_event_ids, d_ylt, ylt_ld: int = 0, flags: int = 0,
                n_trials: Optional[int] = None):
        n = d_trial_offsets.numel() - 1 if n_trials is None else n_trials
        self._check(lib().ara_run(self._ptr, n, _dptr(d_trial_offsets, "torch.uint64"),
                                  _dptr(d_event_ids, "torch.uint32"),
                                  _dptr(d_ylt, "torch.float64"), ylt_ld, flags))

    def ara_run_outputs(self, d_trial_offsets, d_event_ids, d_ylt, d_max_occ=None,
                        d_event_inc=None, flags: int = 0, ylt_ld: int = 0, max_occ_ld: int = 0,
                        event_inc_ld: int = 0):
        o = Outputs(_dptr(d_ylt, "torch.float64"), ylt_ld,
                    None if d_max_occ is None else _dptr(d_max_occ, "torch.float64"), max_occ_ld,
                    None if d_event_inc is None else _dptr(d_event_inc, "torch.float64"),
                    event_inc_ld)
        self._check(lib().ara_run_outputs(self._ptr, d_trial_offsets.numel() - 1,
                                          _dptr(d_trial_offsets, "torch.uint64"),
                                          _dptr(d_event_ids, "torch.uint32"), ctypes.byref(o),
                                          flags))

    def ara_run_host(self, h_trial_offsets, h_event_ids, h_ylt: np.ndarray, ylt_ld: int = 0,
                     flags: int = 0):
        to = _host(h_trial_offsets, np.uint64)
        ev = _host(h_event_ids, np.uint32)
        if not (isinstance(h_ylt, np.ndarray) and h_ylt.dtype == np.float64
                and h_ylt.flags.c_contiguous):
            raise TypeError("h_ylt must be a contiguous float64 numpy array")
        self._check(lib().ara_run_host(self._ptr, to.shape[0] - 1, _hptr(to), _hptr(ev),
                                       _hptr(h_ylt), ylt_ld, flags))

    def ara_ep_curve(self, d_row, d_curve):
        """F4 exceedance curve: d_curve = d_row sorted from the largest value down (stream-
        ordered; both 1-D float64 CUDA tensors of the same length)."""
        n = d_row.numel()
        if d_curve.numel() != n:
            raise ValueError("d_curve must have d_row's length")
        self._check(lib().ara_ep_curve(self._ptr, _dptr(d_row, "torch.float64"), n,
                                       _dptr(d_curve, "torch.float64")))

    def ara_synchronize(self):
        self._check(lib().ara_synchronize(self._ptr))

    def ara_metrics(self, d_ylt_row, p: Sequence[float]):
        pp = np.ascontiguousarray(p, dtype=np.float64)
        pml = np.empty(pp.shape[0]); tvar = np.empty(pp.shape[0])
        self._check(lib().ara_metrics(self._ptr, _dptr(d_ylt_row, "torch.float64"),
                                      d_ylt_row.numel(), pp.shape[0], _hptr(pp), _hptr(pml),
                                      _hptr(tvar)))
        return pml, tvar

    def ara_metrics_rows(self, d_rows, p: Sequence[float], n: int = 0, ld: int = 0):
        """PML / TVaR ([rows][n_p] arrays) of every row of a 2-D device tensor in shared passes
        (``n``: entries per row, default the row length; ``ld``: row stride, default the
        tensor's)."""
        pp = np.ascontiguousarray(p, dtype=np.float64)
        R = d_rows.shape[0]
        n = n or d_rows.shape[1]
        ld = ld or d_rows.stride(0)
        pml = np.empty((R, pp.shape[0])); tvar = np.empty((R, pp.shape[0]))
        self._check(lib().ara_metrics_rows(self._ptr, _dptr(d_rows, "torch.float64"), R, ld, n,
                                           pp.shape[0], _hptr(pp), _hptr(pml), _hptr(tvar)))
        return pml, tvar

    def ara_portfolio_ylt(self, d_ylt, d_out, ylt_ld: int = 0, flags: int = 0):
        """Per-trial sum over the context's layers (layer order) of a device YLT."""
        n = d_out.numel()
        self._check(lib().ara_portfolio_ylt(self._ptr, _dptr(d_ylt, "torch.float64"), n, ylt_ld,
                                            _dptr(d_out, "torch.float64"), flags))
        return d_out

    def ara_metrics_sharded(self, d_ylt_slice, n_global: int, p: Sequence[float], allreduce):
        """PML / TVaR of a YLT row split over ranks (this rank's slice on the device).
        ``allreduce(tensor)`` must sum a CUDA tensor in place across all ranks (e.g.
        ``torch.distributed.all_reduce``); it is called on this context's stream."""
        import torch
        pp = np.ascontiguousarray(p, dtype=np.float64)
        pml = np.empty(pp.shape[0]); tvar = np.empty(pp.shape[0])
        dev = d_ylt_slice.device if d_ylt_slice.is_cuda else torch.device("cuda", self.device)
        xbuf = torch.zeros(ARA_MAX_P * 256, dtype=torch.int64, device=dev)
        err = []

        def cb(offset, count, is_f64, user):
            try:
                view = xbuf.view(torch.uint8)[offset: offset + 8 * count]
                view = view.view(torch.float64 if is_f64 else torch.int64)
                if self.stream is not None:
                    with torch.cuda.stream(self.stream):
                        allreduce(view)
                else:
                    allreduce(view)
                return 0
            except Exception as exc:  # reported as ARA_ERR_ARG by the library
                err.append(exc)
                return 1

        fn = SHARD_REDUCE(cb)
        st = lib().ara_metrics_sharded(self._ptr, _dptr(d_ylt_slice, "torch.float64") if
                                       d_ylt_slice.numel() else None, d_ylt_slice.numel(),
                                       int(n_global), pp.shape[0], _hptr(pp), _hptr(pml),
                                       _hptr(tvar), xbuf.data_ptr(), xbuf.numel() * 8, fn, None)
        if err:
            raise err[0]
        self._check(st)
        return pml, tvar

    def ara_metrics_host(self, h_ylt_row, p: Sequence[float]):
        row = _host(h_ylt_row, np.float64)
        pp = np.ascontiguousarray(p, dtype=np.float64)
        pml = np.empty(pp.shape[0]); tvar = np.empty(pp.shape[0])
        self._check(lib().ara_metrics_host(self._ptr, _hptr(row), row.shape[0], pp.shape[0],
                                           _hptr(pp), _hptr(pml), _hptr(tvar)))
        return pml, tvar

    def ara_get_info(self) -> Info:
        info = Info()
        self._check(lib().ara_get_info(self._ptr, ctypes.byref(info)))
        return info

    def ara_layer_store_shape(self, layer: int):
        u, w = ctypes.c_uint32(), ctypes.c_uint32()
        self._check(lib().ara_layer_store_shape(self._ptr, layer, ctypes.byref(u),
                                                ctypes.byref(w)))
        return u.value, w.value

    def ara_export_store(self, layer: int, catalogue_size: int):
        u, w = self.ara_layer_store_shape(layer)
        m = np.empty(catalogue_size + 1, dtype=np.uint32)
        r = np.empty((u + 1, w), dtype=np.float64)
        self._check(lib().ara_export_store(self._ptr, layer, _hptr(m), _hptr(r)))
        return m, r

    @property
    def kernel_launches(self) -> int:
        return self.ara_get_info().kernel_launches


def ara_status_string(status: int) -> str:
    return lib().ara_status_string(status).decode()
