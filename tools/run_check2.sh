set -x
timeout 900 python -m pytest tests/test_gpu_v6.py tests/test_gpu_golden.py tests/test_gpu_bounds.py tests/test_gpu_parity.py -x -q > gpurun_out/check2_tests.txt 2>&1
tail -3 gpurun_out/check2_tests.txt
timeout 300 python tools/quick_time.py f32 f64 > gpurun_out/check2_qt.txt 2>&1
cat gpurun_out/check2_qt.txt
