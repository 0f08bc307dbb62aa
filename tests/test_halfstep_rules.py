"""Half-step wavefront rules of the v4 pass kernel (bb_api.cu make_plan,
bb_pass_v4.cuh) pinned at the footprint level: a step (r, j) = phase A (row
reflector + right application, cells rows q..hi x cols p..hi) then phase B
(column reflector + left application, rows p..hi x cols p..ce) (Alg. 2,
P:168-182).  A rule says which progress value of sweep r-1 (2j+1 after A(j),
2j+2 after B(j)) each phase of sweep r waits for.  A rule is valid iff every
pair of phases with intersecting cells is ordered as in sequential order
(then every admitted execution equals the sequential oracle bit for bit; the
whole-step version of that statement is pinned against the oracle itself in
test_oracle_schedule.py).  The kernel uses, by target bandwidth c - t:
  >= 4: A 2j+2, B 2j+3;   2..3: A 2j+2, B 2j+4;   1: A 2j+4, B 2j+5
each strictly weaker than the whole-step distance of reading Q4 (s = 2:
2j+4 / 2j+4, s = 3: 2j+6 / 2j+6), and each minimal in the sense that
tightening it by one half-step breaks it."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import depcheck  # noqa: E402


def rule(a, b):
    return (lambda j, J: 2 * j + a), (lambda j, J: 2 * j + b)


KERNEL = {">=4": (2, 3), "2..3": (2, 4), "1": (4, 5)}


def band_class(c, t):
    d = c - t
    return ">=4" if d >= 4 else ("2..3" if d >= 2 else "1")


CASES = [(40, 6, 2), (50, 8, 3), (45, 10, 4), (60, 5, 3), (60, 6, 3), (70, 8, 6), (60, 4, 3), (70, 8, 7),
         (90, 16, 15), (64, 9, 8)]


@pytest.mark.parametrize("n,c,t", CASES)
def test_kernel_rule_orders_every_conflict(n, c, t):
    a, b = KERNEL[band_class(c, t)]
    assert depcheck.check(n, c, t, *rule(a, b)) == 0


@pytest.mark.parametrize("n,c,t", CASES)
def test_kernel_rule_is_minimal(n, c, t):
    a, b = KERNEL[band_class(c, t)]
    # one half-step less on B (or on A, keeping B >= A) admits a conflicting order
    assert depcheck.check(n, c, t, *rule(a, b - 1)) > 0 or b - 1 < a
    if a > 2:
        assert depcheck.check(n, c, t, *rule(a - 1, b)) > 0


def test_whole_step_distance_of_the_paper_also_valid():
    # s = 3 ("three-cycle separation") for target bandwidth 1, s = 2 otherwise
    assert depcheck.check(60, 4, 3, *rule(6, 6)) == 0
    assert depcheck.check(50, 8, 3, *rule(4, 4)) == 0
