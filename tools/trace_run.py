"""Run one reduction with per-step device timestamps (BB_TRACE_FILE) and
summarise where the time of one pass goes: wait, staging, compute+store+release,
and the sweep-to-sweep handoff latency on the critical path."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768); ap.add_argument("--b", type=int, default=128)
ap.add_argument("--dtype", default="f64"); ap.add_argument("--tw", type=int, default=16)
ap.add_argument("--pass_", type=int, default=0); ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--maxb", type=int, default=0)
a = ap.parse_args()
path = "/tmp/bb_trace.bin"
os.environ["BB_TRACE_FILE"] = path; os.environ["BB_TRACE_PASS"] = str(a.pass_)
import torch, synth, paper_2510_12705_b200 as bb
band = torch.from_numpy(synth.random_band(a.n, a.b, a.dtype, seed=0)).cuda()
cfg = bb.Config(tw=a.tw, threads_per_block=a.threads, max_blocks_per_sm=a.maxb)
t0 = time.time(); bb.band_to_bidiag(band, a.b, cfg=cfg); torch.cuda.synchronize(); print("total s", time.time() - t0)
raw = open(path, "rb").read()
hdr = np.frombuffer(raw[:24], dtype=np.int32); S, J, c, t, s, grid = [int(x) for x in hdr]
T = np.frombuffer(raw[24:], dtype=np.uint64).reshape(S, J, 4).astype(np.int64)
print(f"pass c={c} t={t} s={s} grid={grid} traced sweeps={S} steps/sweep={J}")
valid = T[:, :, 3] > 0
w = (T[:, :, 1] - T[:, :, 0])[valid]; ld = (T[:, :, 2] - T[:, :, 1])[valid]; cs = (T[:, :, 3] - T[:, :, 2])[valid]
print("ns median: wait %d  stage %d  compute+store+release %d  (p90 %d %d %d)" % (
    np.median(w), np.median(ld), np.median(cs), np.percentile(w, 90), np.percentile(ld, 90), np.percentile(cs, 90)))
# handoff: (r-1, min(j+s-1, J-1)) done -> (r, j) wait end
h = []
for r in range(1, S):
    for j in range(J):
        if not valid[r, j]: continue
        jp = min(j + s - 1, J - 1)
        if valid[r - 1, jp]: h.append(T[r, j, 1] - T[r - 1, jp, 3])
h = np.array(h)
print("handoff ns median %d p10 %d p90 %d" % (np.median(h), np.percentile(h, 10), np.percentile(h, 90)))
# per-cycle rate: time for sweep r start
starts = T[:, 0, 1]
d = np.diff(starts[starts > 0])
print("sweep start interval ns median %d (=> per-cycle %.0f ns)" % (np.median(d), np.median(d) / s))
step_time = T[:, :, 3] - T[:, :, 1]
print("step (stage->release) median ns", int(np.median(step_time[valid])))
