"""SVD stage 1 on the device: dense -> upper band by block
Householder (bb_stage1.cu), the "classical block Householder" first stage of
P:308.  Checked against what the mathematics fixes, independent of any
implementation: the band has the singular values of A (numpy SVD of the
dense input) and its Frobenius norm; then the paper's known-spectrum accuracy
protocol with all three stages on the device: A = U diag(S) V^T ->
stage 1 -> stage 2 (band -> bidiagonal) -> stage 3 (singular values) vs S."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _stage1(A, b):
    import torch
    import paper_2510_12705_b200 as bb
    band = bb.dense_to_band(torch.from_numpy(np.ascontiguousarray(A)).cuda(), b)
    torch.cuda.synchronize()
    return band.cpu().numpy()


@pytest.mark.parametrize("n,b", [(1, 4), (2, 1), (64, 8), (300, 32), (777, 64), (1024, 128), (130, 200)])
def test_band_has_the_singular_values_of_A(n, b):
    rng = np.random.default_rng(n + 7 * b)
    A = rng.standard_normal((n, n))
    band = _stage1(A, b)
    beff = min(b, max(n - 1, 1))
    D = synth.band_to_dense(band, b)
    # entries outside the upper band do not exist in the output layout; the
    # band itself carries A's singular values and norm (orthogonal equivalence)
    s_ref = np.linalg.svd(A, compute_uv=False)
    s = np.linalg.svd(D, compute_uv=False)
    nf = np.linalg.norm(A)
    assert np.max(np.abs(s - s_ref)) <= 1e-12 * n * nf
    assert abs(np.linalg.norm(D) - nf) <= 1e-12 * n * nf
    assert beff <= b


def test_fp32():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((500, 500)).astype(np.float32)
    band = _stage1(A, 32)
    s = np.linalg.svd(synth.band_to_dense(band.astype(np.float64), 32), compute_uv=False)
    s_ref = np.linalg.svd(A.astype(np.float64), compute_uv=False)
    assert np.max(np.abs(s - s_ref)) <= 1e-5 * 500 * np.linalg.norm(A.astype(np.float64))


@pytest.mark.parametrize("kind", ["arith", "log", "qcirc"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_known_spectrum_protocol_all_stages_on_device(kind, dtype):
    # singular values prescribed, stage 1 -> 2 -> 3 on the B200, error vs S
    import torch
    import paper_2510_12705_b200 as bb
    n, b = 1024, 32
    S = synth.spectrum(kind, n)
    A = synth.known_spectrum_dense(n, S, seed=11)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    At = torch.from_numpy(A).to(tdt).cuda()
    band = bb.dense_to_band(At, b)
    d, e = bb.band_to_bidiag(band, b)
    s = bb.bidiag_svals(d, e)
    torch.cuda.synchronize()
    err = float(np.max(np.abs(s.cpu().numpy() - S)))
    print(kind, dtype, "max |sigma - S| =", err)
    assert err <= (1e-11 if dtype == "f64" else 1e-4)   # S:437 bounds (||A||_2 = 1)
