"""Per-phase timeline of the register kernel (bb_pass_v2.cuh) from BB_TRACE_FILE (16 slots/step)."""
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
bb.band_to_bidiag(band, a.b, cfg=bb.Config(tw=a.tw, max_blocks_per_sm=a.maxb)); torch.cuda.synchronize()
t0 = time.time(); bb.band_to_bidiag(band, a.b, cfg=bb.Config(tw=a.tw, max_blocks_per_sm=a.maxb)); torch.cuda.synchronize()
print("total s %.3f" % (time.time() - t0))
raw = open(path, "rb").read()
S, J, c, t, s, grid = [int(x) for x in np.frombuffer(raw[:24], dtype=np.int32)]
T = np.frombuffer(raw[24:], dtype=np.uint64).reshape(S, J, 16).astype(np.int64)
print(f"pass c={c} t={t} grid={grid}")
names = {0: "W0start", 1: "W0done", 2: "W1start", 3: "W1done", 4: "A_sync", 5: "A_rel", 6: "B_sync", 7: "B_rel",
         8: "C_start", 9: "C_loaded", 10: "C_rowrefl", 11: "C_rightapply", 12: "C_colrefl", 13: "C_W1", 14: "C_Bstored"}
sel = T[1:min(S, 600), 2:min(J, 60)]       # steady-state region
base = sel[:, :, 8]
ok = (sel[:, :, 7] > 0) & (base > 0)
for k in [0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 11, 12, 13, 14]:
    d = (sel[:, :, k] - base)[ok & (sel[:, :, k] > 0)]
    if d.size: print("%-14s median %7d ns  p10 %7d  p90 %7d" % (names[k], np.median(d), np.percentile(d, 10), np.percentile(d, 90)))
# handoff: predecessor A release (slot 5 of (r-1, j+1)) -> W1 done (slot 3 of (r, j))
h = (sel[1:, :-1, 3] - sel[:-1, 1:, 5])
print("A_rel(r-1,j+1) -> W1done(r,j) median", int(np.median(h)))
h2 = (sel[1:, :, 1] - sel[:-1, :, 7])
print("B_rel(r-1,j) -> W0done(r,j) median", int(np.median(h2)))
st = T[1:min(S, 600), 0, 8]
print("sweep period ns", int(np.median(np.diff(st))))
print("step period ns", int(np.median(np.diff(sel[:, :, 8], axis=1))))
