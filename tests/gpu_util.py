"""Helpers for the GPU parity tests (tolerances of BASELINE.json north_star,
read normwise per DESIGN.md reading Q15)."""
from __future__ import annotations

import numpy as np

import oracle
import synth
from tests.lapack_ref import bidiag_svals

TORCH_DT = {"f16": "float16", "f32": "float32", "f64": "float64"}


def tol(dtype: str, n: int) -> float:
    """Normwise tolerance factor tau: max |x_gpu - x_oracle| <= tau * ||A||_F
    for x in {sigma, |d|, |e|} (north_star: 1e-12 n fp64, 1e-5 n fp32, 5e-2 fp16)."""
    return {"f64": 1e-12 * n, "f32": 1e-5 * n, "f16": 5e-2}[dtype]


def gpu_reduce(band: np.ndarray, b: int, tw=None, cfg=None, batched=False):
    import torch
    import paper_2510_12705_b200 as bb
    t = torch.from_numpy(np.ascontiguousarray(band)).cuda()
    if batched:
        d, e = bb.band_to_bidiag_batched(t, b, tw=tw, cfg=cfg)
    else:
        d, e = bb.band_to_bidiag(t, b, tw=tw, cfg=cfg)
    torch.cuda.synchronize()
    return d.cpu().numpy(), e.cpu().numpy()


def compare(band: np.ndarray, b: int, tw: int, dtype: str, d, e, svals: bool = True):
    """Assert GPU (d, e) agrees with the oracle on the same input bits."""
    n = band.shape[0]
    d0, e0 = oracle.band_to_bidiag(band, b, tw)
    d = np.asarray(d, dtype=np.float64)
    e = np.asarray(e, dtype=np.float64)
    nf = float(np.linalg.norm(band.astype(np.float64)))
    tau = tol(dtype, n)
    errs = {
        "d": float(np.max(np.abs(np.abs(d) - np.abs(d0)), initial=0.0)),
        "e": float(np.max(np.abs(np.abs(e) - np.abs(e0)), initial=0.0)),
    }
    if svals and n > 0:
        errs["sigma"] = float(np.max(np.abs(bidiag_svals(d, e) - bidiag_svals(d0, e0))))
    for k, v in errs.items():
        assert v <= tau * nf, (k, v, tau * nf, dtype, n, b, tw)
    return errs
