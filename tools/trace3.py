"""Per-phase timeline of the multi-sweep kernel (bb_pass_v3.cuh) from BB_TRACE_FILE."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768); ap.add_argument("--b", type=int, default=128)
ap.add_argument("--dtype", default="f64"); ap.add_argument("--tw", type=int, default=16)
ap.add_argument("--pass_", type=int, default=0); ap.add_argument("--maxb", type=int, default=0)
a = ap.parse_args()
path = "/tmp/bb_trace.bin"
os.environ["BB_TRACE_FILE"] = path; os.environ["BB_TRACE_PASS"] = str(a.pass_)
import torch, synth, paper_2510_12705_b200 as bb
band = torch.from_numpy(synth.random_band(a.n, a.b, a.dtype, seed=0)).cuda()
cfg = bb.Config(tw=a.tw, max_blocks_per_sm=a.maxb)
bb.band_to_bidiag(band, a.b, cfg=cfg); torch.cuda.synchronize()
t0 = time.time(); bb.band_to_bidiag(band, a.b, cfg=cfg); torch.cuda.synchronize()
print("total s %.3f" % (time.time() - t0))
raw = open(path, "rb").read()
S, J, c, t, G, grid = [int(x) for x in np.frombuffer(raw[:24], dtype=np.int32)]
T = np.frombuffer(raw[24:], dtype=np.uint64).reshape(S, J, 16).astype(np.int64)
print(f"pass c={c} t={t} G={G} grid={grid}")
names = {0: "wait_start", 1: "A_wait_done", 2: "staged", 3: "A_published", 4: "B_wait_done", 5: "complete",
         6: "rowrefl_done", 7: "rightapply_done", 8: "colrefl_done", 9: "leftapply_done"}
sel = T[G:min(S, 600), 2:min(J, 60)]
base = sel[:, :, 1]
ok = (sel[:, :, 5] > 0) & (base > 0)
for k in [0, 2, 6, 7, 3, 8, 4, 9, 5]:
    okk = ok & (sel[:, :, k] > 0)
    d = (sel[:, :, k] - base)[okk]
    if d.size == 0: continue
    print("%-12s median %7d ns  p10 %7d  p90 %7d" % (names[k], np.median(d), np.percentile(d, 10), np.percentile(d, 90)))
for gi in range(G):
    rows = [r for r in range(G, min(S, 600)) if r % G == gi]
    st = T[rows, 0, 1]
    print("WG %d: sweep-to-sweep (r-1 -> r) A-wait-done lag median %d ns" % (gi, np.median(T[rows, 5:40, 1] - T[np.array(rows) - 1, 5:40, 1])))
st = T[G:min(S, 600), 0, 1]
print("sweep period ns", int(np.median(np.diff(st))))
print("step period ns", int(np.median(np.diff(sel[:, :, 1], axis=1))))
