"""P7: the wavefront schedule the GPU relies on is equivalent to sequential order.

The oracle runs sweeps strictly in order.  The GPU runs a wavefront of
concurrent sweeps behind a dependency distance s ("three-cycle
separation"; reading Q4: s = 2 unless the pass's target bandwidth is 1, then
3).  These tests drive the oracle's step function (bb_oracle.c, one step of
Alg. 2) in the GPU's orders and check:
  * footprints of steps in the same cycle T = s*r + j are disjoint;
  * replaying the cycle schedule, and random orders admitted by the flag rule
    "step (r, j) may start once progress[r-1] >= min(j + s, J_{r-1})",
    is BITWISE equal to the sequential result;
  * the rule is not vacuous: s - 1 produces overlapping footprints.
"""
import random

import numpy as np
import pytest

import oracle
import synth


def footprint(n, c, t, r, j):
    g = oracle.step_geometry(n, c, t, r, j)
    q, p, hi, ce = g
    cells = set()
    for i in range(q, hi + 1):
        for jj in range(p, hi + 1):
            cells.add((i, jj))
    for i in range(p, hi + 1):
        for jj in range(p, ce + 1):
            cells.add((i, jj))
    return cells


def cycle_overlaps(n, c, t, s):
    """Number of cycles whose concurrent steps have intersecting footprints."""
    J = [oracle.sweep_len(n, c, t, r) for r in range(n - 1)]
    T_end = max((s * r + J[r] for r in range(n - 1) if J[r] > 0), default=0)
    bad = 0
    for T in range(T_end):
        seen = set()
        clash = False
        for r in range(n - 1):
            j = T - s * r
            if j < 0:
                break
            if j >= J[r]:
                continue
            fp = footprint(n, c, t, r, j)
            if seen & fp:
                clash = True
            seen |= fp
        bad += clash
    return bad


@pytest.mark.parametrize("n,b,tw", [(48, 8, 3), (40, 6, 2), (60, 12, 5), (50, 10, 9)])
def test_footprints_disjoint_at_minimal_s(n, b, tw):
    for ps in oracle.passes(n, b, tw):
        assert cycle_overlaps(n, ps.c, ps.t, ps.s) == 0
        # and the distance is minimal: s - 1 clashes
        assert cycle_overlaps(n, ps.c, ps.t, ps.s - 1) > 0


def test_target_bandwidth_1_needs_three_cycles():
    # P:155 "as the bandwidth narrows, may also conflict with the third"
    n = 40
    assert cycle_overlaps(n, 4, 3, 2) > 0      # TBW = 1 with s = 2 clashes
    assert cycle_overlaps(n, 4, 3, 3) == 0


def _sequential(band, b, tw):
    o = oracle.Oracle(band, b, tw)
    o.run()
    d, e, st = o.extract(store=True)
    o.close()
    return st


def _replay_cycles(band, b, tw, reverse):
    n = band.shape[0]
    o = oracle.Oracle(band, b, tw)
    for ps in oracle.passes(n, b, tw):
        J = [oracle.sweep_len(n, ps.c, ps.t, r) for r in range(n - 1)]
        T_end = max((ps.s * r + J[r] for r in range(n - 1) if J[r] > 0), default=0)
        for T in range(T_end):
            active = [r for r in range(n - 1) if 0 <= T - ps.s * r < J[r]]
            for r in (reversed(active) if reverse else active):
                o.step(ps.c, ps.t, r, T - ps.s * r)
    _, _, st = o.extract(store=True)
    o.close()
    return st


def _replay_flags(band, b, tw, seed):
    n = band.shape[0]
    rng = random.Random(seed)
    o = oracle.Oracle(band, b, tw)
    for ps in oracle.passes(n, b, tw):
        J = [oracle.sweep_len(n, ps.c, ps.t, r) for r in range(n - 1)]
        prog = [0] * (n - 1)
        remaining = sum(J)
        while remaining:
            ready = []
            for r in range(n - 1):
                j = prog[r]
                if j >= J[r]:
                    continue
                if r == 0 or prog[r - 1] >= min(j + ps.s, J[r - 1]):
                    ready.append(r)
                if r > 0 and prog[r - 1] == 0:
                    break
            r = rng.choice(ready)
            o.step(ps.c, ps.t, r, prog[r])
            prog[r] += 1
            remaining -= 1
    _, _, st = o.extract(store=True)
    o.close()
    return st


@pytest.mark.parametrize("n,b,tw", [(64, 8, 3), (50, 10, 9), (45, 16, 4)])
def test_cycle_schedule_bitwise_equals_sequential(n, b, tw):
    band = synth.random_band(n, b, "f64", seed=21)
    ref = _sequential(band, b, tw)
    assert np.array_equal(_replay_cycles(band, b, tw, reverse=False), ref)
    assert np.array_equal(_replay_cycles(band, b, tw, reverse=True), ref)


@pytest.mark.parametrize("seed", range(3))
def test_flag_rule_random_orders_bitwise_equal(seed):
    n, b, tw = 56, 9, 4
    band = synth.random_band(n, b, "f64", seed=30 + seed)
    ref = _sequential(band, b, tw)
    assert np.array_equal(_replay_flags(band, b, tw, seed), ref)
