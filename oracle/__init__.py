"""CPU fp64 oracle for band -> bidiagonal bulge chasing (arXiv 2510.12705).

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2510_12705_b200`` never imports it, and
the two share no code.

The arithmetic lives in ``bb_oracle.c`` (plain sequential C, fp64, header
cites PAPER.md line by line).  This module only:
  * builds/loads that library (``gcc -O2 -ffp-contract=off``),
  * marshals numpy arrays in and out,
  * enumerates the plan (passes, sweeps, step geometry) in pure Python --
    Alg. 1 with readings Q1-Q3 -- for the schedule pins and the
    algorithmic byte / flop counts of SURVEY §8d.

Every function states the passage it follows.  Nothing here is "parity
unpinned": the pins are in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bb_oracle.c")
_LIB = os.path.join(_HERE, "libbb_oracle.so")
_lib = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile bb_oracle.c into oracle/libbb_oracle.so (portable x86-64, no -march)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off",
               "-fno-fast-math", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def use_native_build(outdir: str, compile: bool = True) -> str | None:
    """bench.py cpu_baseline only: compile the same C source with
    ``-march=native`` into ``outdir`` and load that build instead.
    The arithmetic is unchanged (-ffp-contract=off, no fast-math: gcc may not
    reassociate or contract), only instruction selection.  Returns the flags
    used, or None (the portable build stays loaded)."""
    global _lib
    path = os.path.join(outdir, "libbb_oracle_native.so")
    flags = ["-O2", "-march=native", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off", "-fno-fast-math"]
    try:
        if compile:
            os.makedirs(outdir, exist_ok=True)
            subprocess.check_call(["gcc"] + flags + ["-o", path + ".tmp", _SRC, "-lm"], stderr=subprocess.DEVNULL)
            os.replace(path + ".tmp", path)
        elif not os.path.exists(path):
            return None
    except Exception:
        return None
    _lib = None
    lib(path)
    return " ".join(flags)


def lib(path: str | None = None):
    global _lib
    if _lib is None:
        if path is None:
            build()
        L = ctypes.CDLL(path or _LIB)
        L.oracle_house.argtypes = [_i64, _dp, _dp, _dp, _dp]
        L.oracle_house.restype = None
        L.oracle_num_passes.argtypes = [_i64, _i64, _i64]
        L.oracle_num_passes.restype = _i64
        L.oracle_new.argtypes = [_i64, _i64, _i64, _dp, _i64]
        L.oracle_new.restype = ctypes.c_void_p
        L.oracle_free.argtypes = [ctypes.c_void_p]
        L.oracle_free.restype = None
        L.oracle_step.argtypes = [ctypes.c_void_p, _i64, _i64, _i64, _i64]
        L.oracle_step.restype = ctypes.c_int
        L.oracle_run.argtypes = [ctypes.c_void_p, _i64, ctypes.POINTER(_i64), _dp]
        L.oracle_run.restype = ctypes.c_int
        L.oracle_extract.argtypes = [ctypes.c_void_p, _dp, _dp, _dp]
        L.oracle_extract.restype = None
        L.oracle_store_width.argtypes = [ctypes.c_void_p]
        L.oracle_store_width.restype = _i64
        L.oracle_band_to_bidiag.argtypes = [_i64, _i64, _i64, _dp, _i64, _dp, _dp]
        L.oracle_band_to_bidiag.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ---------------------------------------------------------------------------
# Reflector (Alg. 2 "HH(X)"; dlarfg convention, reading Q7/Q8)
# ---------------------------------------------------------------------------

def house(x):
    """(v, tau, beta) with (I - tau v v^T) x = beta e_1, v[0] = 1."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    v = np.zeros_like(x)
    tau = ctypes.c_double()
    beta = ctypes.c_double()
    lib().oracle_house(len(x), _ptr(x), _ptr(v), ctypes.byref(tau), ctypes.byref(beta))
    return v, tau.value, beta.value


# ---------------------------------------------------------------------------
# Whole reduction and the step-level handle
# ---------------------------------------------------------------------------

class Oracle:
    """Step-level handle over the C oracle (used by the schedule pins, P7)."""

    def __init__(self, band: np.ndarray, b: int, tw: int):
        band64 = np.ascontiguousarray(band, dtype=np.float64)
        self.n, self.ld = band64.shape
        self.b, self.tw = b, tw
        self._band = band64
        self.h = lib().oracle_new(self.n, b, tw, _ptr(band64), self.ld)
        if not self.h:
            raise ValueError("oracle_new: bad arguments")

    def step(self, c: int, t: int, r: int, j: int) -> None:
        if lib().oracle_step(self.h, c, t, r, j) != 0:
            raise RuntimeError("oracle: access outside the band + 2*tw store")

    def run(self, max_steps: int = -1):
        done = _i64()
        elems = ctypes.c_double()
        rc = lib().oracle_run(self.h, max_steps, ctypes.byref(done), ctypes.byref(elems))
        if rc != 0:
            raise RuntimeError("oracle: access outside the band + 2*tw store")
        return done.value, elems.value

    def extract(self, store: bool = False):
        n = self.n
        d = np.zeros(n)
        e = np.zeros(max(n - 1, 0) + 1)
        st = None
        if store:
            w = lib().oracle_store_width(self.h)
            st = np.zeros((max(n, 1), w))
        lib().oracle_extract(self.h, _ptr(d), _ptr(e), _ptr(st) if st is not None else None)
        return d, e[: max(n - 1, 0)], st

    def close(self):
        if self.h:
            lib().oracle_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def band_to_bidiag(band: np.ndarray, b: int, tw: int, store: bool = False):
    """Sequential fp64 reduction.  ``band``: LAPACK upper band, shape (n, ldband),
    any float dtype (widened to fp64, reading Q13).  Returns (d, e) or
    (d, e, store) where store[i, (j - i) + tw] = A[i, j] after the reduction."""
    o = Oracle(band, b, tw)
    try:
        o.run()
        d, e, st = o.extract(store)
    finally:
        o.close()
    return (d, e, st) if store else (d, e)


# ---------------------------------------------------------------------------
# Plan enumeration (Alg. 1 lines 1-10; readings Q1-Q4, Q12)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Pass:
    c: int   # current bandwidth CBW
    t: int   # tilewidth removed in this pass
    s: int   # dependency distance: 3 if target bandwidth c - t == 1 else 2 (Q4)


def passes(n: int, b: int, tw: int):
    """Alg. 1 line 1: c0 = min(b, n-1); while c > 1: t = min(tw, c-1); c -= t."""
    out = []
    if n <= 2 or b <= 1:
        return out
    c = min(b, n - 1)
    while c > 1:
        t = min(tw, c - 1)
        out.append(Pass(c, t, 3 if c - t == 1 else 2))
        c -= t
    return out


def step_geometry(n: int, c: int, t: int, r: int, j: int):
    """(q, p, hi, ce) of step j of sweep r in pass (c, t), or None (reading Q3, Q12)."""
    p = r + (c - t) + j * c
    if p > n - 2:
        return None
    q = r if j == 0 else p - c
    hi = min(p + t, n - 1)
    ce = min(hi + c, n - 1)
    return q, p, hi, ce


def sweep_len(n: int, c: int, t: int, r: int) -> int:
    """J_r = number of steps of sweep r: floor((n-2-(r+c-t))/c)+1, or 0."""
    first = r + c - t
    return 0 if first > n - 2 else (n - 2 - first) // c + 1


def anchors_1indexed(n: int, c: int, t: int, r: int):
    """Anchor rows k of Alg. 1 for sweep r, 1-indexed as in Fig. 2."""
    out = []
    j = 0
    while True:
        g = step_geometry(n, c, t, r, j)
        if g is None:
            return out
        out.append(g[0] + 1)
        j += 1


def workload(n: int, b: int, tw: int, elem_bytes: int):
    """Algorithmic work of SURVEY §8d, by enumeration of every step:
    elements = sum m*((hi-q+1)+(ce-p+1)-m), bytes = 2*elem_bytes*elements (R+W),
    flops = sum 4m(hi-q) + 4m(ce-p) + 6m, critical-path cycles = sum over
    passes of max_r (s*r + J_r) (the kernel-per-cycle schedule T = s*r + j)."""
    steps = 0
    elems = 0
    flops = 0
    crit = 0
    for ps in passes(n, b, tw):
        c, t, s = ps.c, ps.t, ps.s
        last = 0
        for r in range(0, n - 1):
            J = sweep_len(n, c, t, r)
            if J == 0:
                break
            last = max(last, s * r + J)
            for j in range(J):
                q, p, hi, ce = step_geometry(n, c, t, r, j)
                m = hi - p + 1
                elems += m * ((hi - q + 1) + (ce - p + 1) - m)
                flops += 4 * m * (hi - q) + 4 * m * (ce - p) + 6 * m
                steps += 1
        crit += last
    return {"steps": steps, "elements": elems, "bytes": 2 * elem_bytes * elems,
            "flops": flops, "critical_cycles": crit, "passes": len(passes(n, b, tw))}


def occupancy_min_n(cbw: int, alus: int) -> int:
    """Eq. (1): full occupancy needs n / (3 CBW) >= ALUs."""
    return 3 * cbw * alus
