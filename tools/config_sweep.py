"""BASELINE configs 2, 3 and (reduced) 5 on one B200: times, GB/s, matrices/s as JSONL.
usage: python tools/config_sweep.py OUT.jsonl [which=2,3,5]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2510_12705_b200 as bb

out = open(sys.argv[1], "a")
which = (sys.argv[2] if len(sys.argv) > 2 else "2,3,5").split(",")


def timed(n, b, dt, tw, batch=1, maxb=0, G=None, reps=5, warm=2):
    if G is None:
        os.environ.pop("BB_V4_G", None)
    else:
        os.environ["BB_V4_G"] = str(G)
    bands = np.stack([synth.random_band(n, b, dt, seed=0, matrix_id=i) for i in range(batch)])
    t = torch.from_numpy(bands).cuda()
    cfg = bb.Config(tw=tw, max_blocks_per_sm=maxb)
    ws = bb.Workspace(n, b, dt, batch, cfg=cfg)
    st = ws.stats
    f = (lambda: bb.band_to_bidiag_batched(t, b, workspace=ws)) if batch > 1 else \
        (lambda: bb.band_to_bidiag(t[0], b, workspace=ws))
    for _ in range(warm):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    tmed = float(np.median(ts))
    rec = {"n": n, "b": b, "dtype": dt, "tw": tw, "batch": batch, "max_blocks_per_sm": maxb, "G_cap": G,
           "passes": st["passes"], "seconds": tmed, "alg_GBps": st["alg_bytes"] * batch / tmed / 1e9,
           "alg_GFLOPs": st["alg_flops"] * batch / tmed / 1e9, "matrices_per_s": batch / tmed}
    out.write(json.dumps(rec) + "\n"); out.flush()
    print(rec, flush=True)


if "2" in which:
    for dt, tw in (("f64", 16), ("f64", 31), ("f32", 31), ("f32", 16)):
        timed(1024, 32, dt, tw, reps=20, warm=3)
if "3" in which:
    for dt in ("f16", "f32", "f64"):
        for tw in (8, 16, 32, 63):
            for maxb in (0, 1, 2):
                for G in (1, 4):
                    try:
                        timed(8192, 64, dt, tw, maxb=maxb, G=G, reps=3, warm=1)
                    except Exception as ex:  # noqa
                        print("FAIL", dt, tw, maxb, G, ex, flush=True)
if "5" in which:
    for b, tw in ((32, 31), (64, 32), (128, 32), (256, 32), (512, 16)):
        try:
            timed(16384, b, "f64", tw, batch=8, reps=2, warm=1)
        except Exception as ex:  # noqa
            print("FAIL", b, tw, ex, flush=True)
