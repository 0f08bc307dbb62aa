#!/usr/bin/env python
"""Write the full-size golden files of the GPU parity tests (tests/golden/*.npz).

Imports only ``oracle`` (the sequential fp64 CPU reduction, Alg. 1/2 of
PAPER.md), ``synth`` (seeded inputs, no method arithmetic) and the
test-side LAPACK reference for the singular values (DLASQ1 on the oracle's own
bidiagonal).  Nothing here touches the CUDA path: every stored value comes from
the oracle (VERDICT r1 "Next round" item 1; BASELINE.json north_star parity
targets).

Each file holds, for one (n, b, dtype, seed, matrix_id):
  absd, abse   |d|, |e| of the oracle's bidiagonal (unique, reading Q14)
  sigma        singular values of that bidiagonal (descending)
  fro          ||A||_F of the dtype-rounded input
  sha256       of the input bytes (the dtype-rounded LAPACK band), so a test
               can prove it regenerated the same input
  meta         json: n, b, dtype, seed, matrix_id, tw (the oracle's), seconds

    python tools/make_golden.py [--only NAME ...] [--jobs J]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# (name, n, b, dtype, seed, matrix_id, oracle tw)
CASES = [
    # BASELINE config 4: the headline (bench input: seed 0, matrix 0)
    ("c4_n32768_b128_f64_s0_m0", 32768, 128, "f64", 0, 0, 32),
    ("c4_n32768_b128_f32_s0_m0", 32768, 128, "f32", 0, 0, 32),
    # BASELINE config 3 at its stated size
    ("c3_n8192_b64_f64_s0_m0", 8192, 64, "f64", 0, 0, 32),
    ("c3_n8192_b64_f32_s0_m0", 8192, 64, "f32", 0, 0, 32),
    ("c3_n8192_b64_f16_s0_m0", 8192, 64, "f16", 0, 0, 32),
    # BASELINE config 2 (crossover size)
    ("c2_n1024_b32_f64_s0_m0", 1024, 32, "f64", 0, 0, 32),
    ("c2_n1024_b32_f32_s0_m0", 1024, 32, "f32", 0, 0, 32),
]
# BASELINE config 5: 64 x n = 16384, bandwidth sweep, fp64; first and last matrix
for _b in (32, 64, 128, 256, 512):
    for _m in (0, 63):
        CASES.append((f"c5_n16384_b{_b}_f64_s0_m{_m}", 16384, _b, "f64", 0, _m, 32))


def input_sha256(band: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(band).tobytes()).hexdigest()


def make(case):
    import oracle
    import synth
    from tests.lapack_ref import bidiag_svals_dqds
    name, n, b, dtype, seed, mid, tw = case
    band = synth.random_band(n, b, dtype, seed=seed, matrix_id=mid)
    t0 = time.time()
    d, e = oracle.band_to_bidiag(band, b, tw)
    secs = time.time() - t0
    sig = bidiag_svals_dqds(d, e)
    fro = float(np.linalg.norm(band.astype(np.float64)))
    meta = {"n": n, "b": b, "dtype": dtype, "seed": seed, "matrix_id": mid, "tw": tw,
            "oracle_seconds": secs, "generator": "tools/make_golden.py (oracle/ + synth/ only)"}
    np.savez_compressed(os.path.join(GOLDEN, name + ".npz"), absd=np.abs(d), abse=np.abs(e), sigma=sig,
                        fro=np.float64(fro), sha256=np.array(input_sha256(band)), meta=np.array(json.dumps(meta)))
    return name, secs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    a = ap.parse_args()
    cases = [c for c in CASES if not a.only or c[0] in a.only]
    # longest first
    cases.sort(key=lambda c: -(c[1] * c[2] ** 1.2))
    with Pool(a.jobs) as p:
        for name, secs in p.imap_unordered(make, cases):
            print(f"{name}: oracle {secs:.1f} s", flush=True)


if __name__ == "__main__":
    main()
