# per-phase timelines of every pass, fp64 vs fp32 (tools/trace5.py, tools/trace6.py)
set -x
for DT in f64 f32; do
  timeout 300 python tools/trace_run5.py 32768 128 $DT 32 3 > /dev/null 2>&1
  python tools/trace5.py gpurun_out/tr5_${DT}_p0.bin gpurun_out/tr5_${DT}_p1.bin gpurun_out/tr5_${DT}_p2.bin > gpurun_out/tr5_summary_$DT.txt 2>&1
  BB_V6_G=4 timeout 200 python tools/trace_run6.py 32768 128 $DT 32 3 > /dev/null 2>&1
  python tools/trace6.py gpurun_out/tr6_${DT}_n32768.bin > gpurun_out/tr6_summary_$DT.txt 2>&1
done
rm -f gpurun_out/tr5_*.bin gpurun_out/tr6_*.bin
