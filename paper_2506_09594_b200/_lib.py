"""ctypes binding of the C ABI in include/tenrec_b200.h.

The product path has exactly one implementation: the CUDA library built
in-tree (``paper_2506_09594_b200/libtenrec_b200.so``).  If it is missing or a
GPU is not visible, every compute call raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtenrec_b200.so")

F32, F64 = 0, 1
TRANSFORM_KINDS = {"fft": 0, "dct": 1, "explicit": 2}

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

# int (*tr_allreduce_fn)(double* buf, int64_t count, void* stream, void* user)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                ctypes.c_void_p, ctypes.c_void_p)

# the tr_comm collectives of the sharded ADMM
COMM_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)
COMM_ALLTOALL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.c_void_p)
COMM_HALO_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)


class TrComm(ctypes.Structure):
    """struct tr_comm (include/tenrec_b200.h)."""

    _fields_ = [("world", ctypes.c_int), ("rank", ctypes.c_int),
                ("allreduce", COMM_ALLREDUCE_FN), ("alltoall", COMM_ALLTOALL_FN),
                ("halo", COMM_HALO_FN), ("user", ctypes.c_void_p)]


# name -> (restype, argtypes); the list is the contract tests check against the header
SIGNATURES = {
    "tr_version": (ctypes.c_int, []),
    "tr_last_error": (ctypes.c_char_p, []),
    "tr_lrta_workspace": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p, _c_i64p,
                                           _c_i64p]),
    "tr_gnhtsvt_randomized": (ctypes.c_int, [
        ctypes.c_int, _vp, _vp, ctypes.c_int, _c_i64p, _c_i64p, _c_i64p, _c_i64p, ctypes.c_uint64,
        ctypes.c_int, _vp, _c_dp, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
        _vp, _vp, _vp, ctypes.c_int64, _vp]),
    "tr_gnhtsvt_randomized_sharded": (ctypes.c_int, [
        ctypes.c_int, _vp, _vp, ctypes.c_int, _c_i64p, ctypes.c_int64, ctypes.c_int64, _c_i64p,
        _c_i64p, _c_i64p, ctypes.c_uint64, ctypes.c_int, _vp, _c_dp, ctypes.c_int,
        ctypes.c_double, ctypes.c_double, ctypes.c_double, ALLREDUCE_FN, _vp, _vp,
        ctypes.c_int64, _vp]),
    "tr_rsthosvd_bki": (ctypes.c_int, [
        ctypes.c_int, _vp, ctypes.c_int, _c_i64p, _c_i64p, _c_i64p, _c_i64p, ctypes.c_uint64,
        _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]),
    "tr_admm_create": (ctypes.c_int, [
        ctypes.c_int, ctypes.c_int, _c_i64p, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, _c_i64p,
        ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
        _c_i64p, _c_i64p, _c_i64p, ctypes.c_uint64, ctypes.c_int, _vp, _c_dp,
        ctypes.POINTER(ctypes.c_void_p)]),
    "tr_admm_create_sharded": (ctypes.c_int, [
        ctypes.c_int, ctypes.c_int, _c_i64p, ctypes.c_int, _vp, _vp, ctypes.c_int, _c_i64p,
        ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_double,
        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
        _c_i64p, _c_i64p, _c_i64p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
        ctypes.POINTER(TrComm), ctypes.POINTER(ctypes.c_void_p)]),
    "tr_admm_step": (ctypes.c_int, [_vp, _c_dp]),
    "tr_admm_lookahead": (ctypes.c_int, [_vp, ctypes.c_int]),
    "tr_admm_read": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp]),
    "tr_admm_destroy": (ctypes.c_int, [_vp]),
    "tr_admm_stream": (_vp, [_vp]),
    "tr_admm_set_sketch": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p,
                                          _c_i64p, _c_i64p, ctypes.c_double, ctypes.c_int64,
                                          ctypes.c_double, ctypes.c_uint64]),
    "tr_gradsys_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _c_i64p, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_void_p)]),
    "tr_gradsys_solve": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_void_p), _vp, _vp]),
    "tr_gradsys_destroy": (ctypes.c_int, [_vp]),
    "tr_launch_count": (ctypes.c_int64, []),
    "tr_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "tr_profile_timeline": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, _c_dp, _c_dp, _c_i64p,
                                           ctypes.c_int]),
    "tr_profile_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, _c_dp, _c_i64p,
                                       ctypes.c_int]),
    "tr_tucker_create": (ctypes.c_int, [
        ctypes.c_int, _vp, ctypes.c_int, _c_i64p, ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p,
        _c_i64p, _c_i64p, ctypes.c_double, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, _vp,
        ctypes.POINTER(ctypes.c_void_p)]),
    "tr_tucker_info": (ctypes.c_int, [_vp, _c_i64p, _c_i64p, _c_i64p, _c_dp, _c_i64p, _c_i64p,
                                      _c_dp]),
    "tr_tucker_read": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp]),
    "tr_tucker_svt": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _c_dp, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, _vp, _vp]),
    "tr_tucker_destroy": (ctypes.c_int, [_vp]),
    "tr_prox": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, _vp, _vp, ctypes.c_int64, _vp]),
}

_LIB = None


class CudaPathError(RuntimeError):
    """The B200 library is unavailable or a kernel call failed."""


def load(path: str = LIB_PATH):
    """Load the shared library and bind every exported symbol (no GPU needed)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise CudaPathError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def lib():
    """The library, after checking that a CUDA device is visible."""
    import torch

    if not torch.cuda.is_available():
        raise CudaPathError("the tenrec B200 path needs a CUDA device; none is visible")
    return load()


def check(rc: int) -> None:
    if rc != 0:
        msg = _LIB.tr_last_error().decode() if _LIB is not None else "?"
        if rc == 1:
            raise ValueError(msg)
        raise CudaPathError(msg)


def i64(values):
    arr = (ctypes.c_int64 * max(1, len(values)))(*[int(v) for v in values])
    return arr


def stream_ptr(stream=None):
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def profile_read(max_entries: int = 64) -> dict:
    """{category: (total_ms, launches)} of the events recorded since enable."""
    lib = load()
    names = ctypes.create_string_buffer(8192)
    ms = (ctypes.c_double * max_entries)()
    cnt = (ctypes.c_int64 * max_entries)()
    n = lib.tr_profile_read(names, 8192, ms, cnt, max_entries)
    if n < 0:
        check(2)
    cats = names.value.decode().split("\n")[:n]
    return {c: (ms[i], cnt[i]) for i, c in enumerate(cats)}
