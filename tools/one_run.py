"""One reduction (for profiling under ncu): python tools/one_run.py N B DTYPE TW [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2510_12705_b200 as bb
n, b, dt, tw = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
band = torch.from_numpy(synth.random_band(n, b, dt, seed=0)).cuda()
for _ in range(reps):
    d, e = bb.band_to_bidiag(band, b, tw=tw)
torch.cuda.synchronize()
print("ok", float(d[:4].double().abs().sum()))
