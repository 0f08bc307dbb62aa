"""Loader for the oracle-written full-size golden files (tests/golden/*.npz,
written by tools/make_golden.py from oracle/ + synth/ only)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_path(name: str) -> str:
    return os.path.join(GOLDEN, name + ".npz")


def load(name: str) -> dict:
    z = np.load(golden_path(name), allow_pickle=False)
    out = {k: z[k] for k in ("absd", "abse", "sigma")}
    out["fro"] = float(z["fro"])
    out["sha256"] = str(z["sha256"])
    out["meta"] = json.loads(str(z["meta"]))
    return out


def input_sha256(band: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(band).tobytes()).hexdigest()


def tol(dtype: str, n: int) -> float:
    """north_star normwise tolerance factor (reading Q15)."""
    return {"f64": 1e-12 * n, "f32": 1e-5 * n, "f16": 5e-2}[dtype]


def errors(g: dict, d, e, svals=None) -> dict:
    """max |x_gpu - x_golden| for x in {|d|, |e|, sigma}, absolute and / ||A||_F."""
    d = np.abs(np.asarray(d, dtype=np.float64))
    e = np.abs(np.asarray(e, dtype=np.float64))
    out = {"d": float(np.max(np.abs(d - g["absd"]), initial=0.0)),
           "e": float(np.max(np.abs(e - g["abse"]), initial=0.0))}
    if svals is not None:
        out["sigma"] = float(np.max(np.abs(np.asarray(svals) - g["sigma"]), initial=0.0))
    out["fro"] = g["fro"]
    return out
