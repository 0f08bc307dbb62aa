"""B200-native band -> bidiagonal reduction (arXiv 2510.12705, SVD stage 2).

The hot path is CUDA (sm_100a) behind the C ABI of ``include/bandbidiag.h``;
this package is its thin Python binding (ctypes + torch marshalling) plus the
multi-GPU batch driver (``dist``).  See DESIGN.md.
"""
from . import _native
from ._native import (BB_F16, BB_F32, BB_F64, BB_FLAG_NONNEG_OUTPUT, BB_SCHED_AUTO, BB_SCHED_CYCLE,
                      BB_SCHED_FLAGS, BBError, bb_band_to_bidiag, bb_band_to_bidiag_batched,
                      bb_band_to_bidiag_batched_ex, bb_band_to_bidiag_ex, bb_band_to_bidiag_host, bb_launch_count,
                      bb_plan, bb_version, bb_workspace_size, bb_bidiag_svals_batched,
                      bb_bidiag_svals_workspace_size, status_string)
from .api import (Config, Workspace, band_to_bidiag, band_to_bidiag_batched, band_to_bidiag_host, bidiag_svals,
                  dense_to_band, launch_count, plan)

__all__ = [
    "BB_F16", "BB_F32", "BB_F64", "BB_FLAG_NONNEG_OUTPUT", "BB_SCHED_AUTO", "BB_SCHED_CYCLE", "BB_SCHED_FLAGS",
    "BBError", "Config", "Workspace", "band_to_bidiag", "band_to_bidiag_batched", "band_to_bidiag_host",
    "bb_band_to_bidiag", "bb_band_to_bidiag_batched", "bb_band_to_bidiag_batched_ex", "bb_band_to_bidiag_ex",
    "bb_band_to_bidiag_host", "bb_launch_count", "bb_plan", "bb_version", "bb_workspace_size", "launch_count",
    "plan", "status_string", "bidiag_svals", "bb_bidiag_svals_batched", "bb_bidiag_svals_workspace_size", "dense_to_band",
]
