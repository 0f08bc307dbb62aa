"""The segment-ring kernel of the target-bandwidth-1 pass (bb_pass_v6.cuh).

It runs exactly the oracle's arithmetic per step (Alg. 2) with the
paper's three-cycle separation, so its output must be BITWISE
equal to the one-sweep-per-CTA kernel (BB_FLAG_NO_SEGMENT_KERNEL) at every
group size G, ring size and batch interleaving -- any protocol slip (a chunk
loaded before the previous group wrote it, a ring slot reused before its
write-back read it, a progress value published early) changes bits.  Also
checked against the oracle directly."""
import numpy as np
import pytest

import synth
from tests.gpu_util import compare, gpu_reduce

pytestmark = pytest.mark.gpu


def _bb():
    import paper_2510_12705_b200 as bb
    return bb


@pytest.mark.parametrize("G", ["1", "2", "3", "4", "6"])
@pytest.mark.parametrize("dtype,n,b,tw", [("f64", 1025, 32, 32), ("f32", 1400, 32, 32), ("f16", 700, 16, 16),
                                          ("f64", 901, 96, 32)])
def test_v6_bitwise_equals_sweep_kernel(G, dtype, n, b, tw, monkeypatch):
    bb = _bb()
    band = synth.random_band(n, b, dtype, seed=60)
    ref = gpu_reduce(band, b, cfg=bb.Config(tw=tw, no_segment=True))
    monkeypatch.setenv("BB_V6_G", G)
    got = gpu_reduce(band, b, tw=tw)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


@pytest.mark.parametrize("R", ["0", "7", "12"])
def test_v6_ring_sizes_bitwise(R, monkeypatch):
    # BB_V6_R caps the ring (0: default); the smallest legal ring forces the
    # producer to wait for write-backs on almost every chunk
    bb = _bb()
    band = synth.random_band(1300, 32, "f64", seed=61)
    ref = gpu_reduce(band, 32, cfg=bb.Config(tw=32, no_segment=True))
    if R != "0":
        monkeypatch.setenv("BB_V6_R", R)
    monkeypatch.setenv("BB_V6_G", "3")
    got = gpu_reduce(band, 32, tw=32)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_v6_matches_oracle_and_batched(dtype):
    n, b = 1500, 32
    bands = np.stack([synth.random_band(n, b, dtype, seed=62 + m) for m in range(3)])
    d, e = gpu_reduce(bands, b, tw=32, batched=True)
    for m in range(3):
        compare(bands[m], b, 32, dtype, d[m], e[m])
        d1, e1 = gpu_reduce(bands[m], b, tw=32)
        assert np.array_equal(d1, d[m]) and np.array_equal(e1, e[m])
