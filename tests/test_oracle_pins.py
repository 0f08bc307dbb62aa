"""Pins of the CPU oracle against things other than itself.

P1 brute force (dense SVD of A vs SVD of the bidiagonal), P2 exact invariants,
P3 special cases, P4 library routines (LAPACK DGBBRD, dense Golub-Kahan),
P5 paper-printed values (Fig. 2 anchors, Table I), P6 the paper's accuracy
protocol at desk scale, P8 reflector closed forms.  P7 (schedule) lives in
test_oracle_schedule.py.  None of these call the CUDA path.
"""
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests.lapack_ref import bidiag_svals, dgbbrd_de, gk_right_first

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EPS = np.finfo(np.float64).eps


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line)
    return rows


# ---------------------------------------------------------------- P8 reflector
@pytest.mark.parametrize("row", _golden("reflector_examples.txt"))
def test_reflector_closed_forms(row):
    lhs, rhs = row.split("|")
    beta_exp, tau_exp = map(float, lhs.split())
    x = np.array(list(map(float, rhs.split())))
    v, tau, beta = oracle.house(x)
    assert beta == pytest.approx(beta_exp, rel=4 * EPS, abs=0)
    assert tau == pytest.approx(tau_exp, rel=4 * EPS, abs=0)
    assert v[0] == 1.0
    H = np.eye(len(x)) - tau * np.outer(v, v)
    y = H @ x
    assert y[0] == pytest.approx(beta, rel=8 * EPS)
    assert np.all(np.abs(y[1:]) <= 8 * EPS * np.linalg.norm(x))


def test_reflector_properties_random():
    g = np.random.default_rng(5)
    for _ in range(2000):
        m = int(g.integers(2, 40))
        x = g.standard_normal(m) * 10.0 ** g.integers(-200, 200)
        v, tau, beta = oracle.house(x)
        nx = np.linalg.norm(x / np.max(np.abs(x))) * np.max(np.abs(x))
        assert abs(abs(beta) - nx) <= 4 * EPS * nx          # |beta| = ||x||
        assert math.copysign(1.0, beta) == -math.copysign(1.0, x[0] if x[0] != 0 else 1.0)
        assert 1.0 <= tau <= 2.0                                # tau in [1, 2]
        # orthogonality of H = I - tau v v^T: tau (v.v) = 2
        assert tau * (v @ v) == pytest.approx(2.0, rel=1e-13)
        # H x = beta e1 (scaled check, no overflow)
        s = np.max(np.abs(x))
        y = x / s - tau * v * (v @ (x / s))
        assert abs(y[0] - beta / s) <= 16 * EPS
        assert np.all(np.abs(y[1:]) <= 16 * EPS)


def test_reflector_underflow_safe():
    # naive sum of squares underflows to 0 here (1e-170^2 = 0); the scaled
    # norm must still produce a genuine reflector
    x = np.array([1e-170, 3e-170, 4e-170])
    v, tau, beta = oracle.house(x)
    assert tau > 0
    assert beta == pytest.approx(-math.sqrt(26) * 1e-170, rel=1e-14)


# ---------------------------------------------------------------- P1 brute force
@pytest.mark.parametrize("tw", [1, 4, 7])
@pytest.mark.parametrize("seed", range(4))
def test_bruteforce_svd_n64_b8(tw, seed):
    n, b = 64, 8  # BASELINE config 1
    band = synth.random_band(n, b, "f64", seed=seed)
    A = synth.band_to_dense(band, b)
    d, e = oracle.band_to_bidiag(band, b, tw)
    B = np.diag(d) + np.diag(e, 1)
    s_ref = np.linalg.svd(A, compute_uv=False)
    s_got = np.linalg.svd(B, compute_uv=False)
    assert np.max(np.abs(s_ref - s_got)) <= 50 * n * EPS * s_ref[0]


@pytest.mark.parametrize("n,b,tw", [(100, 12, 5), (77, 30, 29), (130, 17, 4), (50, 49, 16), (40, 60, 3)])
def test_bruteforce_svd_shapes(n, b, tw):
    band = synth.random_band(n, b, "f64", seed=11)
    A = synth.band_to_dense(band, b)
    d, e = oracle.band_to_bidiag(band, b, tw)
    s_ref = np.linalg.svd(A, compute_uv=False)
    s_got = bidiag_svals(d, e)
    assert np.max(np.abs(s_ref - s_got)) <= 50 * n * EPS * s_ref[0]


# ---------------------------------------------------------------- P2 invariants
@pytest.mark.parametrize("n,b,tw", [(64, 8, 4), (200, 32, 16), (257, 20, 7), (128, 9, 8)])
def test_exact_invariants(n, b, tw):
    band = synth.random_band(n, b, "f64", seed=3)
    A = synth.band_to_dense(band, b)
    d, e, st = oracle.band_to_bidiag(band, b, tw, store=True)
    # every stored entry other than the diagonal and first superdiagonal is EXACTLY 0
    mask = np.ones_like(st, dtype=bool)
    mask[:, tw] = False        # offset 0
    mask[:, tw + 1] = False    # offset 1
    assert np.count_nonzero(st[mask]) == 0
    # Frobenius norm preserved (orthogonal equivalence)
    fa = np.sum(A * A)
    assert abs(fa - (d @ d + e @ e)) <= 20 * n * EPS * fa
    # d0 = a00 bit for bit: row 0 / column 0 are never hit by a left / right reflector
    assert d[0] == A[0, 0]
    # |e0| = ||A[0, 1..b]||: row 0 changes only through right reflectors
    assert abs(abs(e[0]) - np.linalg.norm(A[0, 1:])) <= 8 * EPS * np.linalg.norm(A[0, 1:])
    # tr((B^T B)^2) = tr((A^T A)^2)
    B = np.diag(d) + np.diag(e, 1)
    t_a = np.sum((A.T @ A) ** 2)
    t_b = np.sum((B.T @ B) ** 2)
    assert abs(t_a - t_b) <= 100 * n * EPS * t_a


def test_log_det_invariant_well_conditioned():
    # |det A| = prod |a_ii| = prod |d_i| (triangular, orthogonal equivalence).
    # Only meaningful when no |d_i| is near eps*||A|| (tiny d_i carry large
    # relative error), so use a diagonally dominant band.
    n, b, tw = 300, 24, 8
    band = synth.random_band(n, b, "f64", seed=8)
    band[:, b] += 3.0 * np.sqrt(b + 1)
    A = synth.band_to_dense(band, b)
    d, e = oracle.band_to_bidiag(band, b, tw)
    assert np.min(np.abs(d)) > 1e-3
    la = np.sum(np.log(np.abs(np.diag(A))))
    lb = np.sum(np.log(np.abs(d)))
    assert abs(la - lb) <= 1e-11 * n


# ---------------------------------------------------------------- P3 special cases
@pytest.mark.parametrize("b", [0, 1])
def test_b_le_1_is_bitwise_passthrough(b):
    n = 50
    band = synth.random_band(n, b, "f64", seed=2)
    d, e = oracle.band_to_bidiag(band, b, 4)
    assert np.array_equal(d, band[:, b])
    if b == 1:
        assert np.array_equal(e, band[1:, 0])
    else:
        assert np.all(e == 0)


def test_tiny_orders():
    for n in (0, 1, 2):
        band = synth.random_band(n, 3, "f64", seed=1, ldband=4)
        d, e = oracle.band_to_bidiag(band, 3, 2)
        assert d.shape == (n,) and e.shape == (max(n - 1, 0),)
        if n >= 1:
            assert d[0] == band[0, 3]
        if n == 2:
            assert d[1] == band[1, 3] and e[0] == band[1, 2]


def test_identity_and_diagonal():
    n, b = 40, 6
    band = np.zeros((n, b + 1))
    band[:, b] = 1.0
    d, e = oracle.band_to_bidiag(band, b, 3)
    assert np.all(d == 1.0) and np.all(e == 0.0)
    band[:, b] = np.arange(1, n + 1)
    d, e = oracle.band_to_bidiag(band, b, 3)
    assert np.array_equal(d, np.arange(1, n + 1, dtype=float)) and np.all(e == 0)


def test_already_bidiagonal_declared_wider_is_unchanged():
    # every reflector has an exactly-zero tail => identity
    n, b = 60, 9
    g = np.random.default_rng(0)
    band = np.zeros((n, b + 1))
    band[:, b] = g.standard_normal(n)
    band[1:, b - 1] = g.standard_normal(n - 1)
    d, e = oracle.band_to_bidiag(band, b, 4)
    assert np.array_equal(d, band[:, b]) and np.array_equal(e, band[1:, b - 1])


# ---------------------------------------------------------------- P4 library routines
@pytest.mark.parametrize("n,b,tw", [(64, 8, 4), (300, 16, 16), (512, 32, 16), (400, 24, 23)])
def test_matches_lapack_dgbbrd(n, b, tw):
    band = synth.random_band(n, b, "f64", seed=7)
    d, e = oracle.band_to_bidiag(band, b, tw)
    d2, e2 = dgbbrd_de(band, b)
    nf = np.linalg.norm(band)
    # |d|, |e| unique (Q14) but ill-conditioned in n: normwise tolerance (Q15)
    assert np.max(np.abs(np.abs(d) - np.abs(d2))) <= 1e-12 * n * nf
    assert np.max(np.abs(np.abs(e) - np.abs(e2))) <= 1e-12 * n * nf
    assert np.max(np.abs(bidiag_svals(d, e) - bidiag_svals(d2, e2))) <= 100 * n * EPS * nf


@pytest.mark.parametrize("n,b,tw", [(48, 8, 3), (64, 12, 11)])
def test_matches_dense_golub_kahan(n, b, tw):
    band = synth.random_band(n, b, "f64", seed=9)
    A = synth.band_to_dense(band, b)
    d, e = oracle.band_to_bidiag(band, b, tw)
    d2, e2, B = gk_right_first(A)
    assert np.max(np.abs(np.abs(d) - np.abs(d2))) <= 1e-12 * np.linalg.norm(A)
    assert np.max(np.abs(np.abs(e) - np.abs(e2))) <= 1e-12 * np.linalg.norm(A)


# ---------------------------------------------------------------- P5 paper values
def test_fig2_anchors():
    rows = [list(map(int, r.split())) for r in _golden("fig2_anchors.txt")]
    for c, t, row1, *anchors in rows:
        got = oracle.anchors_1indexed(40, c, t, row1 - 1)
        assert got[: len(anchors)] == anchors


def test_table1_occupancy():
    for r in _golden("table1_occupancy.txt"):
        name, cbw, alus, min_n = r.split()
        assert oracle.occupancy_min_n(int(cbw), int(alus)) == int(min_n), name


def test_pass_plan_remainder():
    # reading Q2: b=128, tw=16 -> 7 passes of 16 then a last pass with t = 15
    ps = oracle.passes(32768, 128, 16)
    assert [p.c for p in ps] == [128, 112, 96, 80, 64, 48, 32, 16]
    assert [p.t for p in ps] == [16] * 7 + [15]
    assert [p.s for p in ps] == [2] * 7 + [3]
    assert [p.c for p in oracle.passes(8192, 64, 32)] == [64, 32]


def test_workload_counts_match_survey_table():
    # SURVEY §8d "Exact totals" (enumeration of the plan)
    w = oracle.workload(1024, 32, 16, 8)
    assert w["steps"] == 49504 and w["critical_cycles"] == 5077
    assert abs(w["bytes"] / 1e9 - 0.737) < 0.001
    w = oracle.workload(64, 8, 4, 8)
    assert w["steps"] == 760 and w["critical_cycles"] == 301


# ---------------------------------------------------------------- P6 accuracy protocol
@pytest.mark.parametrize("kind", ["arith", "log", "qcirc"])
def test_known_spectrum_fp64(kind):
    n, b, tw = 256, 8, 4   # SPEC acceptance: FP64 < 1e-11 at n=256, bw=8
    sig = synth.spectrum(kind, n)
    A = synth.known_spectrum_dense(n, sig, seed=1)
    Ab = synth.dense_to_upper_band(A, b)
    band = synth.dense_to_band(Ab, b)
    d, e = oracle.band_to_bidiag(band, b, tw)
    s = bidiag_svals(d, e)
    assert np.max(np.abs(s - np.sort(sig)[::-1])) / np.max(sig) < 1e-11


def test_known_spectrum_fp32_input():
    n, b, tw = 256, 8, 4   # FP32 < 1e-4: input rounded to fp32 first
    sig = synth.spectrum("arith", n)
    Ab = synth.dense_to_upper_band(synth.known_spectrum_dense(n, sig, seed=2), b)
    band = synth.dense_to_band(Ab, b, "f32")
    d, e = oracle.band_to_bidiag(band, b, tw)
    s = bidiag_svals(d, e)
    assert np.max(np.abs(s - np.sort(sig)[::-1])) / np.max(sig) < 1e-4


def test_storage_height_never_exceeded_large_tw():
    # reading Q11: fill stays in offsets [-t, c+t]; the oracle flags any access
    # outside its band + 2*tw store (oracle_run returns -2 -> RuntimeError)
    for n, b, tw in [(300, 40, 39), (300, 64, 16), (129, 128, 127)]:
        band = synth.random_band(n, b, "f64", seed=4)
        oracle.band_to_bidiag(band, b, tw)
