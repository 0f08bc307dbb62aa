"""Debug: working band after the first K passes (GPU, BB_DEBUG_PASSES) vs the oracle's
sequential state after the same steps.  usage: python tools/v4debug.py N B DTYPE TW K G"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle, paper_2510_12705_b200 as bb
n, b, dt, tw, K, G = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
os.environ["BB_DEBUG_PASSES"] = str(K)
os.environ["BB_V4_G"] = G
band = synth.random_band(n, b, dt, seed=11)
ws = bb.Workspace(n, b, dt, 1, tw=tw)
bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, workspace=ws)
torch.cuda.synchronize()
W = ws.band_view()[0].double().cpu().numpy()
ku = ws.stats["ku"]
steps = 0
for ps in oracle.passes(n, b, tw)[:K]:
    for r in range(n):
        steps += oracle.sweep_len(n, ps.c, ps.t, r)
o = oracle.Oracle(band, b, tw)
o.run(max_steps=steps)
_, _, st = o.extract(store=True)
A_g = np.zeros((n, n)); A_o = np.zeros((n, n))
for j in range(n):
    for i in range(max(0, j - ku), min(n, j + (W.shape[1] - ku))):
        A_g[i, j] = W[j, ku + i - j]
for i in range(n):
    for j in range(max(0, i - tw), min(n, i + st.shape[1] - tw)):
        A_o[i, j] = st[i, (j - i) + tw]
D = np.abs(A_g - A_o)
print("steps", steps, "max diff", D.max(), "max |A|", np.abs(A_o).max())
bad = np.argwhere(D > 1e-9 * max(1, np.abs(A_o).max()))
print("bad cells", len(bad))
if len(bad):
    order = np.argsort(bad[:, 1] * n + bad[:, 0])
    for i, j in bad[order][:25]:
        print(f"  ({i},{j}) off={j-i} gpu={A_g[i,j]:.6g} oracle={A_o[i,j]:.6g}")
    print("min col", bad[:, 1].min(), "min row", bad[:, 0].min())
