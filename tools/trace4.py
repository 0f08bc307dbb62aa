"""Per-phase timeline of the v4 multi-sweep kernel (bb_pass_v4.cuh) from BB_TRACE_FILE.
usage: python tools/trace4.py [--n N --b B --dtype f64 --tw 16 --pass_ 0 --G g]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768); ap.add_argument("--b", type=int, default=128)
ap.add_argument("--dtype", default="f64"); ap.add_argument("--tw", type=int, default=16)
ap.add_argument("--pass_", type=int, default=0); ap.add_argument("--G", default="")
a = ap.parse_args()
path = "/tmp/bb_trace4.bin"
os.environ["BB_TRACE_FILE"] = path; os.environ["BB_TRACE_PASS"] = str(a.pass_)
if a.G: os.environ["BB_V4_G"] = a.G
import torch, synth, paper_2510_12705_b200 as bb
band = torch.from_numpy(synth.random_band(a.n, a.b, a.dtype, seed=0)).cuda()
bb.band_to_bidiag(band, a.b, tw=a.tw); torch.cuda.synchronize()
raw = open(path, "rb").read()
S, J, c, t, G, grid = [int(x) for x in np.frombuffer(raw[:24], dtype=np.int32)]
T = np.frombuffer(raw[24:], dtype=np.uint64).reshape(S, J, 16).astype(np.int64)
print(f"pass {a.pass_}: c={c} t={t} G={G} grid={grid}")
r_lo, r_hi = 4 * G, min(S, 900)
j_lo, j_hi = 3, min(J, 60)
sel = T[r_lo:r_hi, j_lo:j_hi]
base = sel[:, :, 0]
names = {0: "A_go", 1: "R_done", 2: "A_pub", 3: "B_go", 4: "L_done", 5: "step_pub"}
ok = (sel[:, :, 5] > 0) & (base > 0)
for k in range(6):
    d = (sel[:, :, k] - base)[ok]
    print("WG  %-9s median %7d ns  p10 %7d  p90 %7d" % (names[k], np.median(d), np.percentile(d, 10), np.percentile(d, 90)))
# producer rows (first sweep of each group)
rows = np.array([r for r in range(r_lo, r_hi) if r % G == 0])
P = T[rows, j_lo:j_hi]
prev = T[rows - 1, j_lo:j_hi]      # last sweep of the previous group, same step
prev1 = T[rows - 1, j_lo + 1:j_hi + 1] if j_hi + 1 <= J else None
okp = (P[:, :, 6] > 0) & (prev[:, :, 5] > 0)
def med(x, m):
    x = x[m]
    return "median %7d  p10 %7d  p90 %7d" % (np.median(x), np.percentile(x, 10), np.percentile(x, 90)) if x.size else "-"
print("PROD fill_start - prev step_pub(j)      ", med(P[:, :, 6] - prev[:, :, 5], okp))
print("PROD fillT duration                     ", med(P[:, :, 7] - P[:, :, 6], okp))
print("PROD late fill (8 -> 9)                 ", med(P[:, :, 9] - P[:, :, 8], okp))
if prev1 is not None:
    okq = (P[:, :, 8] > 0) & (prev1[:, :, 2] > 0)
    print("PROD late_go - prev A_pub(j+1)          ", med(P[:, :, 8] - prev1[:, :, 2], okq))

print("WG0 A_go - fillT issued                 ", med(P[:, :, 0] - P[:, :, 7], okp))
print("WG0 B_go - late issued                  ", med(P[:, :, 3] - P[:, :, 9], okp))
print("WG0 A_go - prev group step_pub(j)       ", med(P[:, :, 0] - prev[:, :, 5], okp))
for g in range(1, G):
    rr = rows + g
    W = T[rr, j_lo:j_hi]; Wp = T[rr - 1, j_lo:j_hi]
    m = (W[:, :, 0] > 0) & (Wp[:, :, 5] > 0)
    print(f"WG{g} A_go - WG{g-1} step_pub(j)            ", med(W[:, :, 0] - Wp[:, :, 5], m))
st = T[r_lo:r_hi, 0, 0]
print("sweep period ns", int(np.median(np.diff(st))), " step period ns", int(np.median(np.diff(sel[:, :, 0], axis=1))))
