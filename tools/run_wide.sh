set -x
for W in 0 1; do
  for DT in f64 f32; do
    timeout 200 python -c "
import os, sys; sys.path.insert(0,'.')
if '$W' == '1': os.environ['BB_V5_WIDE'] = '1'
from tools.quick_v5 import time_cfg
print('wide', $W, flush=True)
time_cfg(32768, 128, '$DT', 32, reps=2); time_cfg(8192, 64, '$DT', 32, reps=2)" >> gpurun_out/wide.txt 2>&1
  done
done
grep -v '^+' gpurun_out/wide.txt
