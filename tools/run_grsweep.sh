set -x
for cfg in "f64 2 5" "f64 2 7" "f64 3 7" "f64 3 8" "f64 4 9" "f32 3 7" "f32 4 9" "f32 5 11" "f32 4 13"; do
  set -- $cfg
  BB_V6_G=$2 BB_V6_R=$3 timeout 200 python -c "
import sys; sys.path.insert(0,'.')
from tools.quick_v5 import time_cfg
print('dt $1 G $2 R $3', flush=True)
time_cfg(32768, 128, '$1', 32, reps=2)" >> gpurun_out/grsweep.txt 2>&1
done
grep -v '^+' gpurun_out/grsweep.txt
