"""Out-of-bounds and uninitialised-memory checks of every pass kernel without
compute-sanitizer (disabled on the GPU pool: tests/test_gpu_sanitizer.py skips
there).

* Guard bands: the workspace and the (d, e) outputs are carved out of larger
  buffers whose margins hold a sentinel byte pattern; after the reduction the
  margins must be byte-for-byte unchanged (any global write outside the
  documented buffers -- a wrong ldw, a chunk store past the matrix end, a
  flag index past its pass -- lands in a margin or in another buffer checked
  here), and the read-only input band must be bit-identical.
* Workspace poisoning: the same reduction in a workspace pre-filled with NaN
  bit patterns and in a zeroed one must give bitwise equal (d, e): no kernel
  may read a workspace cell it did not write first (the pack kernel
  initialises the whole working band, bb_api.cu), and the progress flags /
  claim counters are reset stream-ordered by the call itself.
Shapes cover each kernel (unit v5, segment ring v6, one-sweep v4, register
v2, generic), the three dtypes, ragged tails and a batch."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

GUARD = 1 << 20          # bytes of margin on each side
PAT = 0xA5


def _bb():
    import paper_2510_12705_b200 as bb
    return bb


def _guarded(nbytes, fill):
    buf = torch.full((GUARD + ((nbytes + 255) // 256) * 256 + GUARD,), fill, dtype=torch.uint8, device="cuda")
    return buf, buf[GUARD: GUARD + nbytes]


def _margins_ok(buf, nbytes):
    body = ((nbytes + 255) // 256) * 256
    lo, hi = buf[:GUARD], buf[GUARD + nbytes:]
    # bytes of the body past nbytes (alignment padding) are margin too
    assert int((lo != PAT).sum()) == 0, "write below the buffer"
    assert int((hi != PAT).sum()) == 0, f"write past the buffer ({body - nbytes} padding bytes + {GUARD} guard)"


def _run(band_np, b, dtype, cfg, batch, ws_fill):
    bb = _bb()
    tdt = {"f16": torch.float16, "f32": torch.float32, "f64": torch.float64}[dtype]
    es = torch.empty(0, dtype=tdt).element_size()
    n, ld = band_np.shape[-2:]
    band = torch.from_numpy(band_np).cuda().reshape(batch, n, ld).contiguous()
    band_before = band.clone()
    st = bb.plan(n, b, dtype, batch, cfg)
    wsb, ws = _guarded(st["workspace_bytes"], PAT)
    if ws_fill is not None:
        ws.fill_(ws_fill)
    dbuf, dv = _guarded(batch * n * es, PAT)
    ebuf, ev = _guarded(batch * max(n - 1, 1) * es, PAT)
    d = dv.view(tdt).view(batch, n)
    e = ev.view(tdt).view(batch, max(n - 1, 1))
    from paper_2510_12705_b200 import _native as N
    N.bb_band_to_bidiag_batched_ex(n, b, bb.api.bb_dtype(dtype), batch, band.data_ptr(), ld, n * ld,
                                   d.data_ptr(), n, e.data_ptr(), max(n - 1, 1), cfg.c(), ws.data_ptr(),
                                   st["workspace_bytes"], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    _margins_ok(wsb, st["workspace_bytes"])
    _margins_ok(dbuf, batch * n * es)
    _margins_ok(ebuf, batch * max(n - 1, 1) * es)
    assert torch.equal(band.view(torch.uint8), band_before.view(torch.uint8)), "input band modified"
    return d.cpu().clone(), e[:, : n - 1].cpu().clone()


CASES = [
    # (n, b, dtype, tw, batch, cfg kwargs)      kernel(s) exercised
    (777, 128, "f64", 32, 1, {}),              # v5 (3 passes) + v6 c=32
    (1301, 96, "f32", 32, 2, {}),              # v5 + v6, batched, ragged
    (513, 64, "f16", 16, 1, {}),               # v5 MT=17 + v6 c=16, fp16 storage
    (600, 64, "f64", 32, 1, {"no_unit": True}),      # v4 multi-sweep + v6
    (600, 64, "f32", 32, 1, {"no_segment": True}),   # v5 + v4 last pass
    (333, 40, "f64", 7, 1, {}),                # v2 register kernel (odd tilewidth)
    (300, 40, "f32", 16, 1, {"generic": True}),      # generic shared-memory kernel
]


@pytest.mark.parametrize("n,b,dtype,tw,batch,kw", CASES)
def test_guard_bands_and_poisoned_workspace(n, b, dtype, tw, batch, kw):
    bb = _bb()
    cfg = bb.Config(tw=tw, **kw)
    band = np.stack([synth.random_band(n, b, dtype, seed=40 + m) for m in range(batch)])
    d0, e0 = _run(band, b, dtype, cfg, batch, ws_fill=0)
    d1, e1 = _run(band, b, dtype, cfg, batch, ws_fill=0xFF)     # all-ones bytes: NaN in every float format
    d2, e2 = _run(band, b, dtype, cfg, batch, ws_fill=None)     # guard pattern inside too
    for x, y in ((d0, d1), (e0, e1), (d0, d2), (e0, e2)):
        assert torch.equal(x.view(torch.uint8), y.view(torch.uint8))
    assert torch.isfinite(d0.double()).all() and torch.isfinite(e0.double()).all()


@pytest.mark.parametrize("n,b,dtype,tw,kw", [(777, 128, "f64", 32, {}), (901, 64, "f32", 32, {}),
                                             (513, 64, "f16", 16, {}), (600, 64, "f64", 32, {"no_unit": True}),
                                             (333, 40, "f64", 7, {}), (300, 40, "f32", 16, {"generic": True})])
def test_check_zeros_flag(n, b, dtype, tw, kw):
    # BB_FLAG_CHECK_ZEROS: the device-side structural-zero check passes on every
    # kernel family and leaves (d, e) identical to the unchecked call
    bb = _bb()
    from tests.gpu_util import gpu_reduce
    band = synth.random_band(n, b, dtype, seed=44)
    ref = gpu_reduce(band, b, cfg=bb.Config(tw=tw, **kw))
    got = gpu_reduce(band, b, cfg=bb.Config(tw=tw, check_zeros=True, **kw))
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


def test_check_zeros_flag_detects_incomplete_reduction(monkeypatch):
    # only the first of three passes run (debug knob): the band is not bidiagonal
    bb = _bb()
    from paper_2510_12705_b200 import _native as N
    from tests.gpu_util import gpu_reduce
    band = synth.random_band(500, 96, "f64", seed=45)
    monkeypatch.setenv("BB_DEBUG_PASSES", "1")
    with pytest.raises(N.BBError) as ex:
        gpu_reduce(band, 96, cfg=bb.Config(tw=32, check_zeros=True))
    assert ex.value.status == N.BB_ERR_INTERNAL
