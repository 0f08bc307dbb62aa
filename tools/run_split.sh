set -x
for Q in 1 2 4; do
  for DT in f64 f32; do
    BB_V6_SPLIT=$Q timeout 200 python -c "
import sys; sys.path.insert(0,'.')
from tools.quick_v5 import time_cfg
print('split', $Q, flush=True)
time_cfg(32768, 128, '$DT', 32, reps=2)" >> gpurun_out/split.txt 2>&1
  done
done
BB_V6_SPLIT=4 timeout 300 python -m pytest tests/test_gpu_v6.py -q -x > gpurun_out/split_tests.txt 2>&1
tail -2 gpurun_out/split_tests.txt
grep -v '^+' gpurun_out/split.txt
