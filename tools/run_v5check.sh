# v5 change check: headline timings, config-3 timings, unit-kernel tests, per-phase trace of pass 1
set -x
timeout 300 python tools/quick_time.py f64 f32 > gpurun_out/v5check_qt.txt 2>&1
timeout 250 python tools/maxb_sweep.py 8192 64 f64 32 0 >> gpurun_out/v5check_qt.txt 2>&1
timeout 250 python tools/maxb_sweep.py 8192 64 f32 32 0 >> gpurun_out/v5check_qt.txt 2>&1
cat gpurun_out/v5check_qt.txt
timeout 900 python -m pytest tests/test_gpu_v5.py tests/test_gpu_golden.py tests/test_gpu_parity.py -x -q > gpurun_out/v5check_tests.txt 2>&1
tail -3 gpurun_out/v5check_tests.txt
bash tools/run_trace5.sh
