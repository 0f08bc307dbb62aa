# v6 change check: parity tests touching the last pass, headline timings, G sweep
set -x
timeout 600 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py tests/test_gpu_bounds.py -x -q > gpurun_out/v6check_tests.txt 2>&1
tail -3 gpurun_out/v6check_tests.txt
timeout 300 python tools/quick_time.py f64 f32 > gpurun_out/v6check_qt.txt 2>&1
for G in ${GS:-2 3 4}; do
  for DT in f64 f32; do
    BB_V6_G=$G timeout 100 python -c "
import sys; sys.path.insert(0,'.')
from tools.quick_v5 import time_cfg
print('G', $G, flush=True); time_cfg(32768, 128, '$DT', 32, reps=2)" >> gpurun_out/v6check_qt.txt 2>&1
  done
done
cat gpurun_out/v6check_qt.txt
