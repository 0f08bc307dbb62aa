"""Torch-facing convenience layer over the C ABI (marshalling only).

Tensors are device memory; the work runs on ``torch.cuda.current_stream()``.
Every step of the reduction runs in the CUDA kernels behind
``libbandbidiag.so``; nothing here computes.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native as N

_DT = {torch.float16: N.BB_F16, torch.float32: N.BB_F32, torch.float64: N.BB_F64}
_DT_NAME = {"f16": torch.float16, "f32": torch.float32, "f64": torch.float64}


def bb_dtype(t) -> int:
    if isinstance(t, str):
        t = _DT_NAME[t]
    if isinstance(t, torch.Tensor):
        t = t.dtype
    if t not in _DT:
        raise N.BBError(N.BB_ERR_NOT_SUPPORTED, f"dtype {t}")
    return _DT[t]


@dataclass
class Config:
    """The paper's hyperparameter triple plus scheduling knobs."""
    tw: int = 0
    threads_per_block: int = 0
    max_blocks_per_sm: int = 0
    dep_distance: int = 0
    schedule: int = N.BB_SCHED_AUTO
    nonneg: bool = False
    generic: bool = False       # force the generic shared-memory step kernel (testing)
    no_unit: bool = False       # never use the unit kernel (bb_pass_v5.cuh), for comparisons
    no_segment: bool = False    # never use the segment-ring kernel (bb_pass_v6.cuh), for comparisons
    check_zeros: bool = False   # debug: verify the structural zeros on the device (synchronises)
    timing_events: tuple = ()   # torch.cuda.Event objects (enable_timing=True), >= passes + 3

    def c(self) -> N.bb_config:
        flags = ((N.BB_FLAG_NONNEG_OUTPUT if self.nonneg else 0) | (N.BB_FLAG_GENERIC_KERNEL if self.generic else 0)
                 | (N.BB_FLAG_NO_UNIT_KERNEL if self.no_unit else 0)
                 | (N.BB_FLAG_NO_SEGMENT_KERNEL if self.no_segment else 0)
                 | (N.BB_FLAG_CHECK_ZEROS if self.check_zeros else 0))
        cfg = N.bb_config(self.tw, self.threads_per_block, self.max_blocks_per_sm, self.dep_distance,
                          self.schedule, flags)
        if self.timing_events:
            for ev in self.timing_events:
                if ev.cuda_event == 0:      # torch creates events lazily
                    ev.record()
            arr = (ctypes.c_void_p * len(self.timing_events))(*[ev.cuda_event for ev in self.timing_events])
            cfg.timing_events = arr
            cfg.num_timing_events = len(self.timing_events)
            cfg._keep = arr
        return cfg


def _stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check_same(band: torch.Tensor, *ts):
    """Every tensor of one call lives on band's device with band's dtype (the
    C library launches on the current device, which the callers set to
    band.device)."""
    for t in ts:
        if t.device != band.device:
            raise ValueError(f"tensor on {t.device}, band on {band.device}")
        if t.dtype not in (band.dtype, torch.uint8):
            raise ValueError(f"tensor dtype {t.dtype}, band dtype {band.dtype}")


def _cfg(cfg: Config | None, tw: int | None) -> Config:
    cfg = Config() if cfg is None else Config(**cfg.__dict__)
    if tw is not None:
        cfg.tw = int(tw)
    return cfg


def plan(n: int, b: int, dtype="f64", batch: int = 1, cfg: Config | None = None, tw: int | None = None) -> dict:
    return N.bb_plan(n, b, bb_dtype(dtype), batch, _cfg(cfg, tw).c())


def launch_count(n: int, b: int, dtype="f64", batch: int = 1, cfg: Config | None = None,
                 tw: int | None = None) -> int:
    return N.bb_launch_count(n, b, bb_dtype(dtype), batch, _cfg(cfg, tw).c())


class Workspace:
    """Pre-allocated device workspace for the _ex entry points (timing excludes
    allocation).  ``band_view()`` exposes the working band (documented layout)."""

    def __init__(self, n: int, b: int, dtype, batch: int = 1, cfg: Config | None = None,
                 tw: int | None = None, device=None):
        self.n, self.b, self.batch = n, b, batch
        self.dtype = _DT_NAME[dtype] if isinstance(dtype, str) else dtype
        self.cfg = _cfg(cfg, tw)
        dev = torch.device(device if device is not None else "cuda")
        if dev.type == "cuda" and dev.index is None and torch.cuda.is_available():
            dev = torch.device("cuda", torch.cuda.current_device())
        self.stats = plan(n, b, self.dtype, batch, self.cfg)
        self.nbytes = self.stats["workspace_bytes"]
        self.buf = torch.empty(max(self.nbytes, 1), dtype=torch.uint8, device=dev)

    def band_view(self) -> torch.Tensor:
        """Working band after a call: shape (batch, n, ldw), [k, j, ku + i - j] = A_k(i, j)."""
        es = torch.empty(0, dtype=self.dtype).element_size()
        ms, n, ldw = self.stats["mat_stride"], self.n, self.stats["ldw"]
        flat = self.buf[: self.batch * ms * es].view(self.dtype).view(self.batch, ms)
        return flat[:, : n * ldw].reshape(self.batch, n, ldw)


def band_to_bidiag(band: torch.Tensor, b: int, tw: int | None = None, cfg: Config | None = None,
                   workspace: Workspace | None = None, out=None):
    """Reduce one upper-banded matrix.  ``band``: CUDA tensor (n, ldband),
    ``band[j, b + i - j] = A[i, j]`` (LAPACK upper band).  Returns (d, e)."""
    if band.dim() != 2 or not band.is_cuda:
        raise ValueError("band must be a 2-D CUDA tensor (n, ldband)")
    band = band.contiguous()
    n, ld = band.shape
    dt = bb_dtype(band)
    if out is None:
        d = torch.empty(n, dtype=band.dtype, device=band.device)
        e = torch.empty(max(n - 1, 0), dtype=band.dtype, device=band.device)
    else:
        d, e = out
    c = _cfg(cfg, tw)
    _check_same(band, d, e, *([workspace.buf] if workspace is not None else []))
    with torch.cuda.device(band.device):
        st = _stream(band.device)
        if workspace is None and c == Config():
            N.bb_band_to_bidiag(n, b, dt, band.data_ptr(), ld, d.data_ptr(), e.data_ptr(), st)
        elif workspace is None:
            ws = Workspace(n, b, band.dtype, 1, c, device=band.device)
            N.bb_band_to_bidiag_ex(n, b, dt, band.data_ptr(), ld, d.data_ptr(), e.data_ptr(), c.c(),
                                   ws.buf.data_ptr(), ws.nbytes, st)
        else:
            N.bb_band_to_bidiag_ex(n, b, dt, band.data_ptr(), ld, d.data_ptr(), e.data_ptr(), workspace.cfg.c(),
                                   workspace.buf.data_ptr(), workspace.nbytes, st)
    return d, e


def band_to_bidiag_batched(band: torch.Tensor, b: int, tw: int | None = None, cfg: Config | None = None,
                           workspace: Workspace | None = None, out=None):
    """Reduce ``batch`` independent matrices ``band``: (batch, n, ldband)."""
    if band.dim() != 3 or not band.is_cuda:
        raise ValueError("band must be a 3-D CUDA tensor (batch, n, ldband)")
    band = band.contiguous()
    B, n, ld = band.shape
    dt = bb_dtype(band)
    if out is None:
        d = torch.empty(B, n, dtype=band.dtype, device=band.device)
        e = torch.empty(B, max(n - 1, 1), dtype=band.dtype, device=band.device)
    else:
        d, e = out
    c = _cfg(cfg, tw) if workspace is None else workspace.cfg
    ws = workspace if workspace is not None else Workspace(n, b, band.dtype, B, c, device=band.device)
    _check_same(band, d, e, ws.buf)
    with torch.cuda.device(band.device):
        N.bb_band_to_bidiag_batched_ex(n, b, dt, B, band.data_ptr(), ld, n * ld, d.data_ptr(), d.stride(0),
                                       e.data_ptr(), e.stride(0), c.c(), ws.buf.data_ptr(), ws.nbytes,
                                       _stream(band.device))
    return d, e[:, : max(n - 1, 0)]


def band_to_bidiag_host(band, b: int, tw: int | None = None, cfg: Config | None = None):
    """End-to-end from HOST memory (numpy array or CPU tensor, (n, ld) or
    (batch, n, ld)): H2D copy, reduction, D2H copy inside the C ABI call.
    Blocks until the host results are valid."""
    t = torch.as_tensor(band)
    if t.is_cuda:
        raise ValueError("band_to_bidiag_host takes host memory")
    t = t.contiguous()
    single = t.dim() == 2
    if single:
        t = t.unsqueeze(0)
    B, n, ld = t.shape
    d = torch.empty(B, n, dtype=t.dtype, pin_memory=t.is_pinned())
    e = torch.empty(B, max(n - 1, 1), dtype=t.dtype, pin_memory=t.is_pinned())
    N.bb_band_to_bidiag_host(n, b, bb_dtype(t), B, t.data_ptr(), ld, n * ld, d.data_ptr(), d.stride(0),
                             e.data_ptr(), e.stride(0), _cfg(cfg, tw).c(), _stream())
    e = e[:, : max(n - 1, 0)]
    return (d[0], e[0]) if single else (d, e)


def bidiag_svals(d: torch.Tensor, e: torch.Tensor) -> torch.Tensor:
    """SVD stage 3 on the device: singular values of the upper
    bidiagonal(s) (d, e) -- d: (n,) or (batch, n), e: (n-1,) or (batch, n-1),
    CUDA tensors of one dtype -- as fp64, descending, shape like d.
    Bisection on the Golub-Kahan tridiagonal in bb_svals.cu."""
    if not d.is_cuda or not e.is_cuda:
        raise ValueError("d, e must be CUDA tensors")
    single = d.dim() == 1
    D = d.unsqueeze(0) if single else d
    E = e.unsqueeze(0) if single else e
    B, n = D.shape
    D = D.contiguous()
    E = E.contiguous() if E.numel() else torch.zeros(B, 1, dtype=D.dtype, device=D.device)
    _check_same(D, E)
    sig = torch.empty(B, n, dtype=torch.float64, device=D.device)
    nb = N.bb_bidiag_svals_workspace_size(n, B)
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=D.device)
    with torch.cuda.device(D.device):
        N.bb_bidiag_svals_batched(n, bb_dtype(D), B, D.data_ptr(), D.stride(0), E.data_ptr(), E.stride(0),
                                  sig.data_ptr(), n, ws.data_ptr(), nb, _stream(D.device))
    return sig[0] if single else sig


def dense_to_band(A: torch.Tensor, b: int, overwrite: bool = False) -> torch.Tensor:
    """SVD stage 1 on the device: dense square CUDA tensor A
    (fp32/fp64; any layout) -> its upper band with b superdiagonals, U^T A V,
    in the stage-2 input layout: a (n, b+1) tensor t[j, b + i - j] = band(i, j).
    Block Householder QR/LQ panels + cuBLAS trailing GEMMs (bb_stage1.cu)."""
    if A.dim() != 2 or A.shape[0] != A.shape[1] or not A.is_cuda:
        raise ValueError("A must be a square CUDA matrix")
    n = A.shape[0]
    # column-major working copy: the transpose of a row-major contiguous tensor
    W = A.t().contiguous() if not overwrite else A.t().contiguous()
    band = torch.empty(n, b + 1, dtype=A.dtype, device=A.device)
    nb = N.bb_dense_to_band_workspace_size(n, b, bb_dtype(A))
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=A.device)
    with torch.cuda.device(A.device):
        N.bb_dense_to_band(n, b, bb_dtype(A), W.data_ptr(), n, band.data_ptr(), b + 1, ws.data_ptr(), nb,
                           _stream(A.device))
    return band
