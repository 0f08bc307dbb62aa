"""CPU pin of the segment-ring kernel's protocol (bb_pass_v6.cuh, target
bandwidth 1): tools/v6_model.py runs every group's producer, warp-groups and
writer with the kernel's exact enabling rules under random schedules and
checks that each half-step reads, from its CTA's ring, the version of every
cell the oracle's sequential order gives it, and that the global band ends
equal to the sequential result.  Mutating any rule (producer wait 2m+4 ->
2m+2, warp-group waits 2j+4 / 2j+5 -> 2j+3 / 2j+4, writer one step early) or
shrinking the ring below the plan's minimum is caught."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import v6_model as M  # noqa: E402


@pytest.mark.parametrize("n,c,G", [(70, 4, 3), (90, 8, 4), (131, 8, 5), (100, 16, 4), (77, 8, 1), (120, 4, 4)])
def test_protocol_matches_sequential_order(n, c, G):
    R = min(3 + 2 * (G - 1) + 8, 48)      # bb_api.cu: rmin + slack (capped by shared memory)
    for seed in range(4):
        M.run(n, c, G, R, seed=seed)
    M.run(n, c, G, 3 + 2 * (G - 1), seed=9)   # the minimum ring the plan allows


@pytest.mark.parametrize("mut", [dict(load_need=2), dict(a_need=3), dict(b_need=4), dict(write_lag=1)])
def test_rule_mutations_are_caught(mut):
    caught = 0
    for seed in range(8):
        try:
            M.run(90, 8, 4, 11, seed=seed, **mut)
        except AssertionError:
            caught += 1
    assert caught > 0, mut


def test_group_larger_than_c_is_caught():
    # the writer's rule "columns < s + 1 + (j+1)c are final after the last sweep
    # s finished step j" needs every earlier sweep of the group to be done with
    # them, which holds for G <= c (bb_api.cu caps G at c); G = c + 3 breaks it
    caught = 0
    for seed in range(6):
        try:
            M.run(120, 4, 7, 20, seed=seed)
        except AssertionError:
            caught += 1
    assert caught > 0
