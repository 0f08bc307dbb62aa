#!/usr/bin/env python
"""The paper's accuracy protocol (Fig. 3) at full scale, all three SVD
stages on the B200:

  A = U diag(S) V^T, S prescribed in [0, 1] (arithmetic / logarithmic /
  quarter-circle, synth.spectrum), U, V Haar-like (QR of seeded Gaussian
  matrices, torch/cuSOLVER on the device: the input generator only)
  -> stage 1 (bb_dense_to_band, block Householder) -> stage 2
  (band_to_bidiag, this repo's hot path) -> stage 3 (bidiag_svals)
  -> max_i |sigma_i - S_i| (||A||_2 = 1, so this is the relative error) and
  that error / (n eps).

Writes one JSON line per trial.
    python tools/accuracy_study.py [--sizes 1024 4096 16384] [--trials 30 30 5]
                                   [--b 32] [--dtypes f64 f32] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_12705_b200 as bb  # noqa: E402

EPS = {"f64": 2.220446049250313e-16, "f32": 1.1920929e-07}


def haar(n, gen):
    g = torch.randn(n, n, generator=gen, device="cuda", dtype=torch.float64)
    q, r = torch.linalg.qr(g)
    return q * torch.sign(torch.diagonal(r))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="*", default=[1024, 4096, 16384])
    ap.add_argument("--trials", type=int, nargs="*", default=[30, 30, 5])
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--dtypes", nargs="*", default=["f64", "f32"])
    ap.add_argument("--kinds", nargs="*", default=["arith", "log", "qcirc"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = open(a.out, "a") if a.out else sys.stdout
    for n, T in zip(a.sizes, a.trials):
        for kind in a.kinds:
            S = synth.spectrum(kind, n)
            St = torch.from_numpy(S).cuda()
            for trial in range(T):
                gen = torch.Generator(device="cuda")
                gen.manual_seed(1000 * n + 17 * trial + hash(kind) % 1000)
                U, V = haar(n, gen), haar(n, gen)
                A64 = (U * St) @ V.T
                del U, V
                for dt in a.dtypes:
                    tdt = torch.float64 if dt == "f64" else torch.float32
                    A = A64.to(tdt)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    band = bb.dense_to_band(A, a.b)
                    torch.cuda.synchronize()
                    t1 = time.perf_counter()
                    d, e = bb.band_to_bidiag(band, a.b)
                    torch.cuda.synchronize()
                    t2 = time.perf_counter()
                    s = bb.bidiag_svals(d, e)
                    torch.cuda.synchronize()
                    t3 = time.perf_counter()
                    err = float(torch.max(torch.abs(s - St)))
                    rec = {"n": n, "b": a.b, "dtype": dt, "spectrum": kind, "trial": trial, "max_abs_err": err,
                           "err_over_n_eps": err / (n * EPS[dt]), "stage1_s": t1 - t0, "stage2_s": t2 - t1,
                           "stage3_s": t3 - t2}
                    out.write(json.dumps(rec) + "\n")
                    out.flush()
                    del A, band, d, e, s
                del A64
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
