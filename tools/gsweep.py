"""Per-pass time vs G cap (BB_V4_G) for one workload: python tools/gsweep.py N B DTYPE TW [G ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2510_12705_b200 as bb
n, b, dt, tw = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
Gs = sys.argv[5:] or ["1", "2", "3", "8"]
band = torch.from_numpy(synth.random_band(n, b, dt, seed=0)).cuda()
for rep in range(2):
    for G in Gs:
        os.environ["BB_V4_G"] = G
        P = bb.plan(n, b, dt, tw=tw)["passes"]
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(P + 3)]
        bb.band_to_bidiag(band, b, cfg=bb.Config(tw=tw, timing_events=tuple(evs)))
        torch.cuda.synchronize()
        pm = [round(evs[1 + p].elapsed_time(evs[2 + p]), 1) for p in range(P)]
        print(f"{dt} tw={tw} G<={G}: total {evs[0].elapsed_time(evs[P+2]):.1f} ms  passes {pm}", flush=True)
