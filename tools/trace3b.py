"""Per-WG phase durations of the multi-sweep kernel (needs the trace slots of bb_pass_v3.cuh)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768); ap.add_argument("--b", type=int, default=128)
ap.add_argument("--dtype", default="f64"); ap.add_argument("--tw", type=int, default=16)
ap.add_argument("--pass_", type=int, default=0)
a = ap.parse_args()
path = "/tmp/bb_trace.bin"
os.environ["BB_TRACE_FILE"] = path; os.environ["BB_TRACE_PASS"] = str(a.pass_)
import torch, synth, paper_2510_12705_b200 as bb
band = torch.from_numpy(synth.random_band(a.n, a.b, a.dtype, seed=0)).cuda()
bb.band_to_bidiag(band, a.b, tw=a.tw); torch.cuda.synchronize()
t0 = time.time(); bb.band_to_bidiag(band, a.b, tw=a.tw); torch.cuda.synchronize()
print("total s %.3f" % (time.time() - t0))
raw = open(path, "rb").read()
S, J, c, t, G, grid = [int(x) for x in np.frombuffer(raw[:24], dtype=np.int32)]
T = np.frombuffer(raw[24:], dtype=np.uint64).reshape(S, J, 16).astype(np.int64)
print(f"pass c={c} t={t} G={G} grid={grid}")
ph = [("Await", 0, 1), ("fill", 1, 2), ("rowrefl", 2, 6), ("rightapp", 6, 7), ("colrefl", 3, 8),
      ("Bwait", 8, 4), ("leftapp", 4, 9), ("scatter+pub", 9, 5), ("next-start", 5, None)]
for g in range(G):
    rows = np.array([r for r in range(G, min(S, 900)) if r % G == g])
    sel = T[rows][:, 2:min(J, 100)]
    ok = (sel[:, :, 5] > 0) & (sel[:, :, 0] > 0)
    out = []
    for name, s0, s1 in ph:
        if s1 is None:
            d = (sel[:, 1:, 0] - sel[:, :-1, 5])[ok[:, 1:] & ok[:, :-1]]
        else:
            d = (sel[:, :, s1] - sel[:, :, s0])[ok]
        out.append("%s %5d" % (name, np.median(d)))
    print("WG%d: " % g + " | ".join(out))
# lag between consecutive sweeps at same step (A-wait done)
sel = T[G:min(S, 900), 2:min(J, 100), 1]
print("sweep lag (A-wait-done) median ns", int(np.median(np.diff(sel, axis=0))))
print("step period median ns", int(np.median(np.diff(sel, axis=1))))
