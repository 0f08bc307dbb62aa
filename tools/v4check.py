"""v4 multi-sweep kernel: bitwise agreement across G (warp-groups per CTA), parity vs the oracle,
and timings of the headline sizes.  usage: python tools/v4check.py [quick]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle, paper_2510_12705_b200 as bb
from tests.gpu_util import compare


def run(band, b, tw, G, cfg=None):
    if G is None:
        os.environ.pop("BB_V4_G", None)
    else:
        os.environ["BB_V4_G"] = str(G)
    t = torch.from_numpy(band).cuda()
    d, e = bb.band_to_bidiag(t, b, tw=tw, cfg=cfg)
    torch.cuda.synchronize()
    return d.cpu().numpy(), e.cpu().numpy()


for (n, b, dt, tw) in [(700, 64, "f64", 16), (2000, 128, "f64", 16), (1500, 96, "f32", 32), (1200, 64, "f16", 32),
                       (1100, 128, "f64", 32), (2500, 128, "f32", 16)]:
    band = synth.random_band(n, b, dt, seed=11)
    res = {}
    for G in (0, 1, 2, 3, 4, None):
        try:
            res[G] = run(band, b, tw, G)
        except Exception as ex:  # noqa
            print("FAIL", n, b, dt, tw, G, ex, flush=True)
    ref = res.get(0)
    same = {G: bool(np.array_equal(res[G][0], res[1][0]) and np.array_equal(res[G][1], res[1][1])) for G in res if G != 0}
    t0 = time.time()
    try:
        errs = compare(band, b, tw, dt, *res[None], svals=False)
        ok = "ok"
    except AssertionError as ex:
        errs, ok = str(ex), "PARITY-FAIL"
    try:
        errs1 = compare(band, b, tw, dt, *res[1], svals=False)
    except AssertionError as ex:
        errs1 = "PARITY-FAIL " + str(ex)
    print(f"n={n} b={b} {dt} tw={tw}: bitwise-vs-G1 {same} {ok} {errs} G1 {errs1} (oracle {time.time()-t0:.1f}s)",
          flush=True)
os.environ.pop("BB_V4_G", None)
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    sys.exit(0)
for (n, b, dt, tw, G) in [(32768, 128, "f64", 16, None), (32768, 128, "f64", 16, 1), (32768, 128, "f64", 16, 2),
                          (32768, 128, "f64", 32, None), (32768, 128, "f32", 32, None), (32768, 128, "f32", 16, None)]:
    if G is None:
        os.environ.pop("BB_V4_G", None)
    else:
        os.environ["BB_V4_G"] = str(G)
    band = torch.from_numpy(synth.random_band(n, b, dt, seed=0)).cuda()
    st = bb.plan(n, b, dt, tw=tw)
    ws = bb.Workspace(n, b, dt, 1, tw=tw)
    bb.band_to_bidiag(band, b, workspace=ws)
    torch.cuda.synchronize()
    P = st["passes"]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(P + 3)]
    d, e = bb.band_to_bidiag(band, b, cfg=bb.Config(tw=tw, timing_events=tuple(evs)))
    torch.cuda.synchronize()
    t = evs[0].elapsed_time(evs[P + 2]) / 1e3
    pm = [round(evs[1 + p].elapsed_time(evs[2 + p]), 1) for p in range(P)]
    print(f"{dt} n={n} b={b} tw={tw} G={G}: {t:.3f} s  {st['alg_bytes']/t/1e9:.0f} GB/s  pass ms {pm}", flush=True)
