import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2510_12705_b200 as bb
n, b, tw, dt = 100, 4, 3, sys.argv[1] if len(sys.argv) > 1 else "f32"
band = synth.random_band(n, b, dt, seed=1)
ps = oracle.passes(n, b, tw)[0]
for T in range(0, 60):
    os.environ["BB_DEBUG_MAX_CYCLES"] = str(T)
    ws = bb.Workspace(n, b, dt, 1, cfg=bb.Config(tw=tw, schedule=bb.BB_SCHED_CYCLE))
    t = torch.from_numpy(band).cuda()
    bb.band_to_bidiag(t, b, workspace=ws); torch.cuda.synchronize()
    W = ws.band_view()[0].double().cpu().numpy(); ku = ws.stats["ku"]
    o = oracle.Oracle(band, b, tw)
    J = [oracle.sweep_len(n, ps.c, ps.t, r) for r in range(n - 1)]
    for TT in range(T):
        for r in range(n - 1):
            j = TT - ps.s * r
            if 0 <= j < J[r]: o.step(ps.c, ps.t, r, j)
    _, _, st = o.extract(store=True)
    # compare: st[i, (j-i)+tw] vs W[j, ku+i-j]
    err = 0; where = None
    for i in range(n):
        for off in range(-tw, b + tw + 1):
            j = i + off
            if 0 <= j < n:
                a = st[i, off + tw]; g = W[j, ku + i - j]
                if abs(a - g) > err: err = abs(a - g); where = (i, j)
    print(T, err, where, flush=True)
    if err > 1e-3: break
