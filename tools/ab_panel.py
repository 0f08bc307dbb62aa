"""Scratch A/B: v5 fp32 register panel (default build) vs the shared-memory
panel (BB_LIB_PATH build with -DBB_V5_REG_PANEL=0): bitwise equality of d, e
on several shapes (fp32 and fp16) + headline timings."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

def child(out):
    sys.path.insert(0, ROOT)
    import torch, synth
    import paper_2510_12705_b200 as bb
    res = {}
    for dt, n, b, tw in (("f32", 1500, 128, 32), ("f32", 3000, 96, 32), ("f16", 1400, 64, 32), ("f32", 2049, 64, 16),
                         ("f64", 1500, 128, 32), ("f64", 2049, 64, 16)):
        band = torch.from_numpy(synth.random_band(n, b, dt, seed=77)).cuda()
        d, e = bb.band_to_bidiag(band, b, tw=tw)
        torch.cuda.synchronize()
        res[f"{dt}_{n}_{b}_{tw}_d"] = d.float().cpu().numpy()
        res[f"{dt}_{n}_{b}_{tw}_e"] = e.float().cpu().numpy()
    np.savez(out, **res)
    from tools.quick_v5 import time_cfg
    time_cfg(32768, 128, "f32", 32, reps=2)
    time_cfg(32768, 128, "f64", 32, reps=2)

if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(sys.argv[1]); sys.exit(0)
    env = dict(os.environ)
    subprocess.run([sys.executable, __file__, "/tmp/ab_new.npz"], env=env, check=True)
    for tag in ("oldpanel", "regf64"):
        env["BB_LIB_PATH"] = os.path.join(ROOT, "tools", "ablib", f"libbandbidiag_{tag}.so")
        print("=== lib", tag, flush=True)
        subprocess.run([sys.executable, __file__, f"/tmp/ab_{tag}.npz"], env=env, check=True)
        a, b = np.load("/tmp/ab_new.npz"), np.load(f"/tmp/ab_{tag}.npz")
        for k in a.files:
            print(tag, k, "bitwise" if np.array_equal(a[k], b[k]) else "DIFF max %g" % np.max(np.abs(a[k] - b[k])))
