import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2510_12705_b200 as bb
n, b, tw, dt = 1024, 32, 16, "f32"
band = synth.random_band(n, b, dt, seed=1)
def run(T):
    os.environ["BB_DEBUG_MAX_CYCLES"] = str(T)
    ws = bb.Workspace(n, b, dt, 1, cfg=bb.Config(tw=tw, schedule=bb.BB_SCHED_CYCLE))
    t = torch.from_numpy(band).cuda()
    bb.band_to_bidiag(t, b, workspace=ws); torch.cuda.synchronize()
    return ws.band_view()[0].double().cpu().numpy(), ws.stats["ku"]
# note: BB_DEBUG_MAX_CYCLES caps every pass; find first pass-1 cycle with non-finite / huge values
lo, hi = 0, 4000
W, ku = run(hi)
print("final finite:", np.isfinite(W).all(), np.nanmax(np.abs(W)))
while hi - lo > 1:
    mid = (lo + hi) // 2
    W, ku = run(mid)
    bad = (~np.isfinite(W)).any() or np.nanmax(np.abs(W)) > 1e6
    if bad: hi = mid
    else: lo = mid
print("first bad cycle", hi)
W0, _ = run(lo); W1, _ = run(hi)
print("max before", np.max(np.abs(W0)), "min nonzero", np.min(np.abs(W0[W0 != 0])))
idx = np.argwhere(~np.isfinite(W1) | (np.abs(W1) > 1e6))[:10]
print(idx)
for (j, rho) in idx[:3]:
    i = j + rho - ku
    print("cell i,j", i, j, "before", W0[j, rho], "after", W1[j, rho])
