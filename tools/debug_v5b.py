import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_2510_12705_b200 as bb
from tests.gpu_util import gpu_reduce
n, b, tw = 300, 64, 16
band = synth.random_band(n, b, "f64", seed=50)
d, e = gpu_reduce(band, b, tw=tw)
print("gpu_reduce nan d", np.isnan(d).sum(), "nan e", np.isnan(e).sum(), "inf", np.isinf(d).sum(), np.isinf(e).sum())
ws = bb.Workspace(n, b, "f64", 1, cfg=bb.Config(tw=tw))
d2, e2 = bb.band_to_bidiag(torch.from_numpy(band).cuda(), b, workspace=ws)
torch.cuda.synchronize()
d2 = d2.cpu().numpy(); e2 = e2.cpu().numpy()
print("ws nan", np.isnan(d2).sum(), np.isnan(e2).sum(), "equal", np.array_equal(d, d2, equal_nan=True))
W = ws.band_view()[0].double().cpu().numpy(); ku = ws.stats["ku"]
print("W diag equals d2", np.array_equal(W[:, ku], d2), "nan in W", np.isnan(W).sum())
d0, e0 = oracle.band_to_bidiag(band, b, tw)
print("err", np.nanmax(np.abs(np.abs(d2) - np.abs(d0))), np.nanmax(np.abs(np.abs(e2) - np.abs(e0))))
idx = np.where(~np.isfinite(d))[0]; print("bad d idx", idx[:20]); idx = np.where(~np.isfinite(e))[0]; print("bad e idx", idx[:20])
