# fp32 segment-ring group size at the config sizes (default G vs capped)
set -x
for G in 0 4 5 7; do
  BB_V6_G=$G timeout 200 python -c "
import os, sys; sys.path.insert(0,'.')
if os.environ['BB_V6_G'] == '0': del os.environ['BB_V6_G']
from tools.quick_v5 import time_cfg
print('G', $G, flush=True)
time_cfg(1024, 32, 'f32', 32, reps=3); time_cfg(8192, 64, 'f32', 32, reps=2); time_cfg(32768, 128, 'f32', 32, reps=2)
time_cfg(16384, 128, 'f32', 32, reps=2)" >> gpurun_out/g6f32.txt 2>&1
done
cat gpurun_out/g6f32.txt
