# v5 change check: unit-kernel tests, WA trace, headline timings
set -x
timeout 600 python -m pytest tests/test_gpu_v5.py tests/test_gpu_golden.py tests/test_gpu_bounds.py -x -q > gpurun_out/v5check_tests.txt 2>&1
tail -3 gpurun_out/v5check_tests.txt
bash tools/run_trace5.sh
timeout 300 python tools/quick_time.py f64 f32 > gpurun_out/v5check_qt.txt 2>&1
cat gpurun_out/v5check_qt.txt gpurun_out/tr5_wa.txt
