"""Per-pass time vs max_blocks_per_sm (the paper's "Max blocks"): python tools/maxb_sweep.py N B DTYPE TW [maxb ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2510_12705_b200 as bb
n, b, dt, tw = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
mbs = [int(x) for x in sys.argv[5:]] or [0, 1, 2, 3]
band = torch.from_numpy(synth.random_band(n, b, dt, seed=0)).cuda()
for rep in range(2):
    for mb in mbs:
        P = bb.plan(n, b, dt, tw=tw)["passes"]
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(P + 3)]
        bb.band_to_bidiag(band, b, cfg=bb.Config(tw=tw, max_blocks_per_sm=mb, timing_events=tuple(evs)))
        torch.cuda.synchronize()
        pm = [round(evs[1 + p].elapsed_time(evs[2 + p]), 1) for p in range(P)]
        print(f"{dt} tw={tw} maxb={mb}: total {evs[0].elapsed_time(evs[P+2]):.1f} ms  passes {pm}", flush=True)
