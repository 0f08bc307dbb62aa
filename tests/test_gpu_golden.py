"""Full-size parity: the CUDA path at BASELINE.json's own sizes against the
oracle's results stored in tests/golden/ (tools/make_golden.py: oracle/ +
synth/ only, nothing from the CUDA path).  Element-wise on |d|, |e| and the
singular values, within the north_star tolerances (normwise, reading Q15),
in the launch configuration bench.py times (default config, _ex workspace)."""
import numpy as np
import pytest

import synth
from tests.golden_util import errors, input_sha256, load, tol
from tests.lapack_ref import bidiag_svals_dqds

pytestmark = pytest.mark.gpu


def _run_single(band, b, dtype):
    import torch
    import paper_2510_12705_b200 as bb
    n = band.shape[0]
    ws = bb.Workspace(n, b, dtype, 1)
    d, e = bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, workspace=ws)
    torch.cuda.synchronize()
    return d.double().cpu().numpy(), e.double().cpu().numpy()


@pytest.mark.parametrize("name,n,b,dtype", [
    ("c4_n32768_b128_f64_s0_m0", 32768, 128, "f64"),     # BASELINE config 4, the headline
    ("c4_n32768_b128_f32_s0_m0", 32768, 128, "f32"),
    ("c3_n8192_b64_f64_s0_m0", 8192, 64, "f64"),         # config 3 at its stated size
    ("c3_n8192_b64_f32_s0_m0", 8192, 64, "f32"),
    ("c3_n8192_b64_f16_s0_m0", 8192, 64, "f16"),
    ("c2_n1024_b32_f64_s0_m0", 1024, 32, "f64"),         # config 2
    ("c2_n1024_b32_f32_s0_m0", 1024, 32, "f32"),
])
def test_golden_single(name, n, b, dtype):
    g = load(name)
    band = synth.random_band(n, b, dtype, seed=g["meta"]["seed"], matrix_id=g["meta"]["matrix_id"])
    assert input_sha256(band) == g["sha256"], "regenerated input differs from the golden's input"
    d, e = _run_single(band, b, dtype)
    sv = bidiag_svals_dqds(d, e) if dtype != "f16" else None
    err = errors(g, d, e, sv)
    lim = tol(dtype, n) * g["fro"]
    print(name, {k: v / g["fro"] for k, v in err.items() if k != "fro"})
    for k in ("d", "e", "sigma"):
        if k in err:
            assert err[k] <= lim, (name, k, err[k], lim)


@pytest.mark.parametrize("b", [32, 64, 128, 256, 512])
def test_golden_config5_batched(b):
    # BASELINE config 5 (64 x n = 16384, fp64): matrices 0 and 63 through the
    # batched entry point (their sweeps interleaved in the same launches)
    import torch
    import paper_2510_12705_b200 as bb
    n = 16384
    gs = [load(f"c5_n16384_b{b}_f64_s0_m{m}") for m in (0, 63)]
    bands = np.stack([synth.random_band(n, b, "f64", seed=0, matrix_id=m) for m in (0, 63)])
    for k, g in enumerate(gs):
        assert input_sha256(bands[k]) == g["sha256"]
    ws = bb.Workspace(n, b, "f64", 2)
    d, e = bb.band_to_bidiag_batched(torch.from_numpy(bands).cuda(), b, workspace=ws)
    torch.cuda.synchronize()
    d = d.cpu().numpy()
    e = e.cpu().numpy()
    for k, g in enumerate(gs):
        err = errors(g, d[k], e[k], bidiag_svals_dqds(d[k], e[k]))
        lim = tol("f64", n) * g["fro"]
        print(b, k, {kk: v / g["fro"] for kk, v in err.items() if kk != "fro"})
        for kk in ("d", "e", "sigma"):
            assert err[kk] <= lim, (b, k, kk, err[kk], lim)
