"""ctypes binding of include/bandbidiag.h (argument marshalling only).

Every entry point of the C ABI is exposed under the same name.  The shared
library is built in-tree by ``__graft_entry__.build()`` into
``paper_2510_12705_b200/lib/libbandbidiag.so``; if it is missing, importing
the compute entry points raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libbandbidiag.so")
# A/B experiments only: load another build of the same library
if os.environ.get("BB_LIB_PATH"):
    LIB_PATH = os.environ["BB_LIB_PATH"]

BB_F16, BB_F32, BB_F64 = 0, 1, 2
BB_SUCCESS = 0
BB_ERR_INVALID_VALUE = 1
BB_ERR_NOT_SUPPORTED = 2
BB_ERR_OUT_OF_MEMORY = 3
BB_ERR_CUDA = 4
BB_ERR_INTERNAL = 5
BB_SCHED_AUTO, BB_SCHED_FLAGS, BB_SCHED_CYCLE = 0, 1, 2
BB_FLAG_NONNEG_OUTPUT = 0x1
BB_FLAG_GENERIC_KERNEL = 0x2
BB_FLAG_NO_UNIT_KERNEL = 0x4
BB_FLAG_NO_SEGMENT_KERNEL = 0x8
BB_FLAG_CHECK_ZEROS = 0x10

EXPORTED = [
    "bb_band_to_bidiag", "bb_band_to_bidiag_batched", "bb_band_to_bidiag_ex",
    "bb_band_to_bidiag_batched_ex", "bb_band_to_bidiag_host", "bb_workspace_size", "bb_plan",
    "bb_launch_count", "bb_status_string", "bb_version", "bb_bidiag_svals", "bb_bidiag_svals_batched",
    "bb_bidiag_svals_workspace_size", "bb_dense_to_band", "bb_dense_to_band_workspace_size",
]


class bb_config(ctypes.Structure):
    _fields_ = [("tw", ctypes.c_int32), ("threads_per_block", ctypes.c_int32),
                ("max_blocks_per_sm", ctypes.c_int32), ("dep_distance", ctypes.c_int32),
                ("schedule", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("timing_events", ctypes.POINTER(ctypes.c_void_p)), ("num_timing_events", ctypes.c_int32)]


class bb_plan_stats(ctypes.Structure):
    _fields_ = [("passes", ctypes.c_int64), ("steps", ctypes.c_int64),
                ("critical_cycles", ctypes.c_int64), ("alg_elements", ctypes.c_double),
                ("alg_bytes", ctypes.c_double), ("alg_flops", ctypes.c_double),
                ("tw", ctypes.c_int32), ("threads_per_block", ctypes.c_int32),
                ("ldw", ctypes.c_int64), ("ku", ctypes.c_int64), ("mat_stride", ctypes.c_int64),
                ("workspace_bytes", ctypes.c_size_t)]


class BBError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)}")


_lib = None
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_cfgp = ctypes.POINTER(bb_config)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py` (build()) first; "
                              "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        i = ctypes.c_int
        L.bb_band_to_bidiag.argtypes = [_i64, _i64, i, _vp, _i64, _vp, _vp, _vp]
        L.bb_band_to_bidiag_batched.argtypes = [_i64, _i64, i, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp]
        L.bb_band_to_bidiag_ex.argtypes = [_i64, _i64, i, _vp, _i64, _vp, _vp, _cfgp, _vp, ctypes.c_size_t, _vp]
        L.bb_band_to_bidiag_batched_ex.argtypes = [_i64, _i64, i, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _i64,
                                                   _cfgp, _vp, ctypes.c_size_t, _vp]
        L.bb_band_to_bidiag_host.argtypes = [_i64, _i64, i, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _cfgp, _vp]
        L.bb_workspace_size.argtypes = [_i64, _i64, i, _i64, _cfgp, ctypes.POINTER(ctypes.c_size_t)]
        L.bb_plan.argtypes = [_i64, _i64, i, _i64, _cfgp, ctypes.POINTER(bb_plan_stats)]
        L.bb_launch_count.argtypes = [_i64, _i64, i, _i64, _cfgp, ctypes.POINTER(_i64)]
        L.bb_bidiag_svals.argtypes = [_i64, i, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
        L.bb_bidiag_svals_batched.argtypes = [_i64, i, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, ctypes.c_size_t,
                                              _vp]
        L.bb_bidiag_svals_workspace_size.argtypes = [_i64, _i64, ctypes.POINTER(ctypes.c_size_t)]
        L.bb_dense_to_band.argtypes = [_i64, _i64, i, _vp, _i64, _vp, _i64, _vp, ctypes.c_size_t, _vp]
        L.bb_dense_to_band_workspace_size.argtypes = [_i64, _i64, i, ctypes.POINTER(ctypes.c_size_t)]
        L.bb_status_string.argtypes = [i]
        L.bb_status_string.restype = ctypes.c_char_p
        L.bb_version.argtypes = []
        L.bb_version.restype = ctypes.c_int32
        for name in EXPORTED:
            if name not in ("bb_status_string", "bb_version"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().bb_status_string(int(s)).decode()


def _check(s: int, where: str):
    if s != BB_SUCCESS:
        raise BBError(s, where)


def _cfg(cfg):
    return ctypes.byref(cfg) if cfg is not None else None


# ---- same-name thin wrappers (raw pointers as ints) -------------------------
def bb_band_to_bidiag(n, b, dtype, band, ldband, d_out, e_out, stream=0):
    _check(lib().bb_band_to_bidiag(n, b, dtype, band, ldband, d_out, e_out, stream), "bb_band_to_bidiag")


def bb_band_to_bidiag_batched(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d, e_out, stride_e,
                              stream=0):
    _check(lib().bb_band_to_bidiag_batched(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d,
                                           e_out, stride_e, stream), "bb_band_to_bidiag_batched")


def bb_band_to_bidiag_ex(n, b, dtype, band, ldband, d_out, e_out, cfg, workspace, workspace_bytes, stream=0):
    _check(lib().bb_band_to_bidiag_ex(n, b, dtype, band, ldband, d_out, e_out, _cfg(cfg), workspace,
                                      workspace_bytes, stream), "bb_band_to_bidiag_ex")


def bb_band_to_bidiag_batched_ex(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d, e_out, stride_e,
                                 cfg, workspace, workspace_bytes, stream=0):
    _check(lib().bb_band_to_bidiag_batched_ex(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d,
                                              e_out, stride_e, _cfg(cfg), workspace, workspace_bytes, stream),
           "bb_band_to_bidiag_batched_ex")


def bb_band_to_bidiag_host(n, b, dtype, batch, band_host, ldband, stride_band, d_host, stride_d, e_host, stride_e,
                           cfg=None, stream=0):
    _check(lib().bb_band_to_bidiag_host(n, b, dtype, batch, band_host, ldband, stride_band, d_host, stride_d,
                                        e_host, stride_e, _cfg(cfg), stream), "bb_band_to_bidiag_host")


def bb_workspace_size(n, b, dtype, batch=1, cfg=None) -> int:
    out = ctypes.c_size_t()
    _check(lib().bb_workspace_size(n, b, dtype, batch, _cfg(cfg), ctypes.byref(out)), "bb_workspace_size")
    return out.value


def bb_plan(n, b, dtype, batch=1, cfg=None) -> dict:
    st = bb_plan_stats()
    _check(lib().bb_plan(n, b, dtype, batch, _cfg(cfg), ctypes.byref(st)), "bb_plan")
    return {f: getattr(st, f) for f, _ in bb_plan_stats._fields_}


def bb_launch_count(n, b, dtype, batch=1, cfg=None) -> int:
    out = _i64()
    _check(lib().bb_launch_count(n, b, dtype, batch, _cfg(cfg), ctypes.byref(out)), "bb_launch_count")
    return out.value


def bb_version() -> int:
    return lib().bb_version()


def bb_bidiag_svals_workspace_size(n, batch=1) -> int:
    out = ctypes.c_size_t()
    _check(lib().bb_bidiag_svals_workspace_size(n, batch, ctypes.byref(out)), "bb_bidiag_svals_workspace_size")
    return out.value


def bb_bidiag_svals_batched(n, dtype, batch, d, stride_d, e, stride_e, sigma, stride_sigma, workspace,
                            workspace_bytes, stream):
    _check(lib().bb_bidiag_svals_batched(n, dtype, batch, d, stride_d, e, stride_e, sigma, stride_sigma,
                                         workspace, workspace_bytes, stream), "bb_bidiag_svals_batched")


def bb_dense_to_band_workspace_size(n, b, dtype) -> int:
    out = ctypes.c_size_t()
    _check(lib().bb_dense_to_band_workspace_size(n, b, dtype, ctypes.byref(out)), "bb_dense_to_band_workspace_size")
    return out.value


def bb_dense_to_band(n, b, dtype, A, lda, band, ldband, workspace, workspace_bytes, stream):
    _check(lib().bb_dense_to_band(n, b, dtype, A, lda, band, ldband, workspace, workspace_bytes, stream),
           "bb_dense_to_band")
