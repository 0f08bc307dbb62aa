"""CPU pins of the unit kernel's reordering (reading Q20) and of its
inter-group wait rule -- dense fp64 replays, independent of the CUDA path:

* unit order (all G row reflectors of step j, then all G column reflectors)
  vs the oracle's sequential order: same |d|, |e| and singular values to
  rounding, structural zeros exact, every unit inside its declared window;
* random interleavings of groups allowed by the closed-form distance give
  results BITWISE equal to the canonical group order;
* for target bandwidth 1 no lock-step unit order is valid (the structure
  breaks), which is why that pass keeps the sequential order (v6);
* the (a0, b0) half-unit rule bb_api.cu uses is safe on the kernel's exact
  load / write-back rectangles (tools/v5_rules.py hazard search)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import v5_proto as P  # noqa: E402
import v5_rules as R  # noqa: E402


def _band(n, b, seed):
    rng = np.random.default_rng(seed)
    return np.triu(np.tril(rng.standard_normal((n, n)), b))


@pytest.mark.parametrize("n,b,tw,gmax", [(60, 8, 2, 3), (90, 12, 4, 5), (97, 16, 4, 8), (130, 24, 8, 6),
                                         (150, 32, 8, 24)])
def test_unit_order_equals_sequential_to_rounding(n, b, tw, gmax):
    A0 = _band(n, b, n + b)
    Gf = lambda c, t: max(1, min(gmax, c - t))  # noqa: E731  (G <= c - t)
    S = P.seq_reduce(A0, b, tw)
    U = P.unit_reduce(A0, b, tw, Gf, check_windows=True)
    for M in (S, U):
        off = M - np.diag(np.diag(M)) - np.diag(np.diag(M, 1), 1)
        assert np.all(off == 0)
    assert np.max(np.abs(np.abs(np.diag(S)) - np.abs(np.diag(U)))) < 1e-10
    assert np.max(np.abs(np.abs(np.diag(S, 1)) - np.abs(np.diag(U, 1)))) < 1e-10
    sv = np.linalg.svd(A0, compute_uv=False)
    assert np.max(np.abs(np.linalg.svd(U, compute_uv=False) - sv)) < 1e-11
    for trial in range(2):
        Rr = P.unit_reduce(A0, b, tw, Gf, order="random", rng=np.random.default_rng(trial))
        assert np.array_equal(Rr, U)


def test_lockstep_units_break_target_bandwidth_one():
    n, c = 80, 8
    A0 = _band(n, c, 5)
    for G in (2, 3):
        A = A0.copy()
        t = c - 1
        ns = n - 1
        for k in range((ns + G - 1) // G):
            j = 0
            while True:
                live = [g for g in range(G) if k * G + g < ns and P.geo(n, c, t, k * G + g, j) is not None]
                if not live:
                    break
                for g in live:
                    P.op_A(A, n, c, t, k * G + g, j)
                for g in live:
                    P.op_B(A, n, c, t, k * G + g, j)
                j += 1
        off = A - np.diag(np.diag(A)) - np.diag(np.diag(A, 1), 1)
        assert np.max(np.abs(off)) > 1e-3   # fill-in left behind: not a valid reduction


def _rule(c, t, G):
    # bb_api.cu (unit kernel): (a0, b0, b0 while the predecessor is in its last unit)
    if 3 * G <= c - t:
        return 2, 3, 4
    if 2 * G <= c - t:
        return 2, 4, 4
    return 4, 5, 5


@pytest.mark.parametrize("c,t,G", [(32, 16, 8), (48, 16, 16), (24, 8, 8), (40, 16, 16), (64, 32, 16), (64, 32, 8),
                                   (128, 32, 32), (96, 32, 16), (36, 12, 8), (50, 14, 12)])
def test_inter_group_rule_is_safe(c, t, G):
    a0, b0, b0t = _rule(c, t, G)
    n = 8 * c + 10 * G + 7
    for nn in (n, n + c // 2 + 1, n + G + 2, n + c + 5):
        assert R.safe(nn, c, t, G, a0, b0, kmax=3, tail_b0=b0t)


@pytest.mark.parametrize("c,t,G", [(96, 32, 32), (64, 32, 16), (128, 32, 32)])
def test_shorter_rules_are_unsafe(c, t, G):
    # the hazard search is not vacuous: one half-step less than the rule used fails
    a0, b0, b0t = _rule(c, t, G)
    n = 8 * c + 10 * G + 7
    res = [R.safe(nn, c, t, G, a0, b0 - 1, kmax=3, tail_b0=b0t) and R.safe(nn, c, t, G, a0, b0, kmax=3, tail_b0=b0t - 1)
           for nn in (n, n + c // 2 + 1, n + c + 5)]
    assert not all(res)
