set -x
timeout 200 python tools/trace_run6.py 32768 128 f64 32 3 > gpurun_out/tr6run.txt 2>&1
timeout 200 python tools/trace_run6.py 32768 128 f32 32 3 >> gpurun_out/tr6run.txt 2>&1
python tools/trace6.py gpurun_out/tr6_f64_n32768.bin gpurun_out/tr6_f32_n32768.bin > gpurun_out/tr6_summary.txt 2>&1
rm -f gpurun_out/tr6_*.bin
