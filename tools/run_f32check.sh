set -x
timeout 300 python tools/quick_time.py f32 f64 > gpurun_out/f32check_qt.txt 2>&1
timeout 250 python tools/maxb_sweep.py 8192 64 f32 32 0 1 >> gpurun_out/f32check_qt.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_v5.py tests/test_gpu_golden.py tests/test_gpu_parity.py -x -q > gpurun_out/f32check_tests.txt 2>&1
tail -3 gpurun_out/f32check_tests.txt
cat gpurun_out/f32check_qt.txt
