"""Small reductions through every pass kernel, for compute-sanitizer runs
(tests/test_gpu_sanitizer.py): unit kernel (v5) at G = 8 / 16, segment-ring
kernel (v6) at G = 1 / 2 / 4, the one-sweep-per-CTA kernel (v4), the
register kernel (v2) and the generic kernel, fp64/fp32/fp16, plus stage 3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_12705_b200 as bb  # noqa: E402


def run(band, b, cfg):
    d, e = bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, cfg=cfg)
    torch.cuda.synchronize()
    return d.double().cpu().numpy(), e.double().cpu().numpy()


def main_sync():
    """Kernels without mbarrier rings (synccheck models every mbarrier phase as
    consumed by a wait; the v4/v6 counters let waiters skip phases, see
    tools/ubench/sync_mb.cu): the unit kernel v5 (first pass only, via
    BB_DEBUG_PASSES), the register kernel v2, the generic kernel, stage 3."""
    n, b = int(os.environ.get("SAN_N", "200")), 64
    for dtype in ("f64", "f32", "f16"):
        band = synth.random_band(n, b, dtype, seed=3)
        os.environ["BB_DEBUG_PASSES"] = "1"
        for G5 in ("8", "16"):
            os.environ["BB_V5_G"] = G5
            run(band, b, bb.Config(tw=32))
        os.environ.pop("BB_V5_G", None)
        os.environ.pop("BB_DEBUG_PASSES", None)
        run(band, b, bb.Config(tw=16, generic=True))
        run(band, b, bb.Config(tw=8, no_unit=True, no_segment=True))  # t + 1 = 9: register kernel v2
    d, e = run(synth.random_band(n, b, "f64", seed=3), b, bb.Config(tw=16, generic=True))
    bb.bidiag_svals(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    torch.cuda.synchronize()
    print("san_run ok")


def main():
    if os.environ.get("SAN_MODE") == "sync":
        return main_sync()
    n, b = int(os.environ.get("SAN_N", "200")), 64
    ref = None
    for dtype in ("f64", "f32", "f16"):
        band = synth.random_band(n, b, dtype, seed=3)
        cfgs = [bb.Config(tw=32), bb.Config(tw=16), bb.Config(tw=32, no_unit=True),
                bb.Config(tw=32, no_unit=True, no_segment=True), bb.Config(tw=16, generic=True)]
        for G5 in ("8", "16"):
            os.environ["BB_V5_G"] = G5
            run(band, b, bb.Config(tw=32))
        os.environ.pop("BB_V5_G", None)
        for G6 in ("1", "2", "4"):
            os.environ["BB_V6_G"] = G6
            run(band, b, bb.Config(tw=32))
        os.environ.pop("BB_V6_G", None)
        for c in cfgs:
            d, e = run(band, b, c)
            if dtype == "f64":
                ref = d if ref is None else ref
    d, e = run(synth.random_band(n, b, "f64", seed=3), b, bb.Config(tw=32))
    bb.bidiag_svals(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    torch.cuda.synchronize()
    print("san_run ok")


if __name__ == "__main__":
    main()
