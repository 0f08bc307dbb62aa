"""SVD stage 3 on the device (the paper uses LAPACK BDSDC
on (d, e)): singular values of the bidiagonal by bisection on
the Golub-Kahan tridiagonal (bb_svals.cu), compared with LAPACK DLASQ1 (dqds,
a different algorithm) on the same (d, e); normwise tolerances (reading
Q15).  The last test runs stage 2 AND stage 3 on the device at the headline
size and compares with the oracle's golden singular values."""
import numpy as np
import pytest

import synth
from tests.golden_util import input_sha256, load, tol
from tests.lapack_ref import bidiag_svals_dqds

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16


def _dev_svals(d, e, dtype="float64"):
    import torch
    import paper_2510_12705_b200 as bb
    D = torch.tensor(np.asarray(d), dtype=getattr(torch, dtype)).cuda()
    E = torch.tensor(np.asarray(e), dtype=getattr(torch, dtype)).cuda()
    s = bb.bidiag_svals(D, E)
    torch.cuda.synchronize()
    return s.cpu().numpy()


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 500, 3001])
def test_random_bidiagonal_matches_dqds(n):
    rng = np.random.default_rng(100 + n)
    d = rng.standard_normal(n)
    e = rng.standard_normal(n - 1)
    s = _dev_svals(d, e)
    ref = bidiag_svals_dqds(d, e)
    nrm = np.sqrt(np.sum(d * d) + np.sum(e * e))
    assert np.all(np.diff(s) <= 0)                      # descending
    assert np.max(np.abs(s - ref)) <= 16 * EPS * max(nrm, 1e-300) * max(1.0, np.log2(n + 1))


def test_special_cases():
    # identity: sigma = 1; a zero superdiagonal splits the problem; zeros on the diagonal
    assert np.allclose(_dev_svals(np.ones(7), np.zeros(6)), 1.0, atol=4 * EPS)
    d = np.array([3.0, -4.0, 0.0, 2.0, 1e-3])
    e = np.array([0.0, 1.5, 0.0, -2.0])
    ref = bidiag_svals_dqds(d, e)
    assert np.max(np.abs(_dev_svals(d, e) - ref)) <= 32 * EPS * np.linalg.norm(np.r_[d, e])
    # graded: singular values over 12 orders of magnitude (absolute, normwise accuracy)
    g = np.logspace(0, -12, 40)
    ref = bidiag_svals_dqds(g, 0.5 * g[1:])
    assert np.max(np.abs(_dev_svals(g, 0.5 * g[1:]) - ref)) <= 32 * EPS * np.linalg.norm(g)


@pytest.mark.parametrize("dtype", ["float32", "float16"])
def test_low_precision_inputs_are_widened(dtype):
    rng = np.random.default_rng(7)
    d = rng.standard_normal(300).astype(dtype)
    e = rng.standard_normal(299).astype(dtype)
    ref = bidiag_svals_dqds(d.astype(np.float64), e.astype(np.float64))
    s = _dev_svals(d, e, dtype)
    assert np.max(np.abs(s - ref)) <= 64 * EPS * np.linalg.norm(np.r_[d, e].astype(np.float64))


def test_batched_equals_single():
    import torch
    import paper_2510_12705_b200 as bb
    rng = np.random.default_rng(9)
    D = torch.tensor(rng.standard_normal((5, 400))).cuda()
    E = torch.tensor(rng.standard_normal((5, 399))).cuda()
    S = bb.bidiag_svals(D, E)
    for k in range(5):
        assert torch.equal(S[k], bb.bidiag_svals(D[k], E[k]))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_headline_stage2_and_stage3_on_device(dtype):
    # BASELINE config 4: band -> bidiagonal -> singular values, all on the
    # device, against the oracle's golden singular values (oracle bidiagonal +
    # dqds), north_star tolerance
    import torch
    import paper_2510_12705_b200 as bb
    n, b = 32768, 128
    g = load(f"c4_n{n}_b{b}_{dtype}_s0_m0")
    band = synth.random_band(n, b, dtype, seed=0)
    assert input_sha256(band) == g["sha256"]
    d, e = bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, workspace=bb.Workspace(n, b, dtype, 1))
    s = bb.bidiag_svals(d, e)
    torch.cuda.synchronize()
    err = float(np.max(np.abs(s.cpu().numpy() - g["sigma"])))
    print(dtype, "max |sigma - sigma_oracle| / ||A||_F =", err / g["fro"])
    assert err <= tol(dtype, n) * g["fro"]
