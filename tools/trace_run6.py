import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2510_12705_b200 as bb
n, b, dt, tw, p = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
band = torch.from_numpy(synth.random_band(n, b, dt, seed=0)).cuda()
bb.band_to_bidiag(band, b, tw=tw); torch.cuda.synchronize()
os.environ["BB_TRACE_FILE"] = f"gpurun_out/tr6_{dt}_n{n}.bin"; os.environ["BB_TRACE_PASS"] = str(p)
bb.band_to_bidiag(band, b, tw=tw); torch.cuda.synchronize()
