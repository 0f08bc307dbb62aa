"""The unit kernel (bb_pass_v5.cuh): G consecutive sweeps advanced one step at
a time, all G row reflectors of the step before its G column reflectors
(exactly commuting reorder, reading Q20).

* against the oracle at every group size G and at the edges of the plan
  (first unit j = 0, clipped last units, sweeps that end inside a group);
* against the sweep-per-warp-group kernels (BB_FLAG_NO_UNIT_KERNEL): both
  within tolerance of the oracle (not bitwise: the order differs);
* deterministic: run to run, over occupancy caps and batched interleaving
  (the progress-flag protocol orders every conflicting pair)."""
import numpy as np
import pytest

import synth
from tests.gpu_util import compare, gpu_reduce

pytestmark = pytest.mark.gpu


def _bb():
    import paper_2510_12705_b200 as bb
    return bb


@pytest.mark.parametrize("G", ["8", "16", "24", "32"])
@pytest.mark.parametrize("dtype,n,b,tw", [("f64", 1500, 128, 32), ("f32", 1333, 96, 32), ("f64", 1200, 64, 16),
                                          ("f16", 900, 64, 16), ("f32", 2049, 128, 16)])
def test_v5_group_sizes_match_oracle(G, dtype, n, b, tw, monkeypatch):
    monkeypatch.setenv("BB_V5_G", G)
    band = synth.random_band(n, b, dtype, seed=50)
    d, e = gpu_reduce(band, b, tw=tw)
    compare(band, b, tw, dtype, d, e, svals=(dtype != "f16"))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_v5_vs_sweep_kernels(dtype):
    bb = _bb()
    n, b, tw = 1700, 128, 32
    band = synth.random_band(n, b, dtype, seed=51)
    d5, e5 = gpu_reduce(band, b, tw=tw)
    d4, e4 = gpu_reduce(band, b, cfg=bb.Config(tw=tw, no_unit=True))
    compare(band, b, tw, dtype, d5, e5)
    compare(band, b, tw, dtype, d4, e4)


@pytest.mark.parametrize("n", [130, 131, 257, 300, 301, 515])
def test_v5_small_and_ragged(n):
    # few groups, units clipped at the matrix end, last group partly empty
    b, tw = 64, 16
    band = synth.random_band(n, b, "f64", seed=52)
    d, e = gpu_reduce(band, b, tw=tw)
    compare(band, b, tw, "f64", d, e)


@pytest.mark.parametrize("maxb", [1, 2])
def test_v5_deterministic(maxb):
    bb = _bb()
    band = synth.random_band(3000, 128, "f64", seed=53)
    ref = gpu_reduce(band, 128, tw=32)
    again = gpu_reduce(band, 128, tw=32)
    capped = gpu_reduce(band, 128, cfg=bb.Config(tw=32, max_blocks_per_sm=maxb))
    for got in (again, capped):
        assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


def test_v5_batched_bitwise_equals_single():
    n, b, B = 1100, 128, 3
    bands = synth.random_band_batch(B, n, b, "f64", seed=54)
    d, e = gpu_reduce(bands, b, batched=True)
    for k in range(B):
        ds, es = gpu_reduce(bands[k], b)
        assert np.array_equal(d[k], ds) and np.array_equal(e[k], es), k


def test_v5_structural_zeros_exact():
    import torch
    bb = _bb()
    n, b = 2000, 128
    band = synth.random_band(n, b, "f64", seed=55)
    ws = bb.Workspace(n, b, "f64", 1)
    d, e = bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, workspace=ws)
    torch.cuda.synchronize()
    W = ws.band_view()[0].double().cpu().numpy()
    ku = ws.stats["ku"]
    mask = np.ones_like(W, dtype=bool)
    mask[:, ku] = False
    mask[1:, ku - 1] = False
    assert np.count_nonzero(W[mask]) == 0
