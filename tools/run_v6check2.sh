set -x
timeout 300 python tools/quick_time.py f64 f32 > gpurun_out/v6c2.txt 2>&1
for cfg in "f64 4 9" "f64 3 7" "f32 4 13" "f32 5 11"; do
  set -- $cfg
  BB_V6_G=$2 BB_V6_R=$3 timeout 200 python -c "
import sys; sys.path.insert(0,'.')
from tools.quick_v5 import time_cfg
print('dt $1 G $2 R $3', flush=True)
time_cfg(32768, 128, '$1', 32, reps=2)" >> gpurun_out/v6c2.txt 2>&1
done
grep -v '^+' gpurun_out/v6c2.txt
timeout 400 python -m pytest tests/test_gpu_v6.py tests/test_gpu_bounds.py -q -x > gpurun_out/v6c2_tests.txt 2>&1; tail -2 gpurun_out/v6c2_tests.txt
