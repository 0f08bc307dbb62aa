"""Time the full reduction (n=32768, b=128) for several dtypes / tilewidths / kernels."""
import os, sys, time, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2510_12705_b200 as bb
n, b = int(os.environ.get("N", 32768)), int(os.environ.get("B", 128))
cases = [x.split(":") for x in sys.argv[1:]] or [("f64", "16", ""), ("f64", "32", "")]
for dt, tw, env in cases:
    for kv in filter(None, env.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    band = torch.from_numpy(synth.random_band(n, b, dt, seed=0)).cuda()
    st = bb.plan(n, b, dt, tw=int(tw))
    ws = bb.Workspace(n, b, dt, 1, tw=int(tw))
    d, e = bb.band_to_bidiag(band, b, workspace=ws); torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        t0 = time.time(); bb.band_to_bidiag(band, b, workspace=ws); torch.cuda.synchronize(); ts.append(time.time() - t0)
    t = min(ts)
    print(f"{dt} tw={tw} {env or '-'}: {t:.3f} s  {st['alg_bytes']/t/1e9:.0f} GB/s  passes={st['passes']}", flush=True)
    for kv in filter(None, env.split(",")):
        del os.environ[kv.split("=")[0]]
