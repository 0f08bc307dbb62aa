"""Scratch GPU check of the unit kernel: small oracle comparisons, then the
headline timing per pass (CUDA events on the launching stream)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth, oracle
import paper_2510_12705_b200 as bb
from tests.gpu_util import compare, gpu_reduce

def run_small():
    for dtype, n, b, tw in [("f64", 300, 64, 16), ("f64", 1500, 128, 32), ("f32", 1333, 96, 32), ("f16", 900, 64, 16)]:
        band = synth.random_band(n, b, dtype, seed=50)
        t0 = time.time()
        d, e = gpu_reduce(band, b, tw=tw)
        errs = compare(band, b, tw, dtype, d, e, svals=(dtype != "f16"))
        print("small", dtype, n, b, tw, errs, "%.2fs" % (time.time() - t0), flush=True)

def time_cfg(n, b, dtype, tw, reps=3, no_unit=False, G=None):
    if G: os.environ["BB_V5_G"] = str(G)
    band = torch.from_numpy(synth.random_band(n, b, dtype, seed=0)).cuda()
    cfg = bb.Config(tw=tw, no_unit=no_unit)
    ws = bb.Workspace(n, b, dtype, 1, cfg=cfg)
    P = ws.stats["passes"]
    d = torch.empty(n, dtype=band.dtype, device="cuda"); e = torch.empty(n - 1, dtype=band.dtype, device="cuda")
    st = torch.cuda.current_stream()
    res = []
    for r in range(reps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(P + 3)]
        c = bb.Config(tw=tw, no_unit=no_unit, timing_events=tuple(evs))
        bb.bb_band_to_bidiag_ex(n, b, bb.api.bb_dtype(dtype), band.data_ptr(), b + 1, d.data_ptr(), e.data_ptr(),
                                c.c(), ws.buf.data_ptr(), ws.nbytes, st.cuda_stream)
        torch.cuda.synchronize()
        passes = [evs[1 + p].elapsed_time(evs[2 + p]) for p in range(P)]
        res.append((evs[0].elapsed_time(evs[P + 2]), passes))
    tot, passes = min(res)
    gb = ws.stats["alg_bytes"] / (tot * 1e-3) / 1e9
    print(f"time n={n} b={b} {dtype} tw={tw} G={G} no_unit={no_unit}: {tot:.1f} ms  passes {['%.1f' % x for x in passes]}  {gb:.0f} GB/s", flush=True)
    if G: del os.environ["BB_V5_G"]
    return d.double().cpu().numpy(), e.double().cpu().numpy()

if __name__ == "__main__":
    run_small()
    for G in (8, 16, 24, 32):
        time_cfg(32768, 128, "f64", 32, G=G)
    d, e = time_cfg(32768, 128, "f64", 32)
    from tests.golden_util import load, errors, tol
    g = load("c4_n32768_b128_f64_s0_m0")
    err = errors(g, d, e)
    print("golden f64", {k: v / g["fro"] for k, v in err.items()}, "tol", tol("f64", 32768))
    d, e = time_cfg(32768, 128, "f32", 32)
    g = load("c4_n32768_b128_f32_s0_m0")
    print("golden f32", {k: v / g["fro"] for k, v in errors(g, d, e).items()})
    time_cfg(32768, 128, "f64", 16)
    time_cfg(8192, 64, "f64", 32); time_cfg(8192, 64, "f32", 32); time_cfg(8192, 64, "f64", 16)
