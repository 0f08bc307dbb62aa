# v5 per-phase trace of passes 0..P-1 and the A write-back cycle breakdown
set -x
timeout 300 python tools/trace_run5.py 32768 128 ${DT:-f64} 32 ${P:-1} > gpurun_out/tr5run.txt 2>&1
python -c "
import sys; sys.path.insert(0,'tools'); import trace5
trace5.summarize('gpurun_out/tr5_${DT:-f64}_p0.bin'); trace5.wa_cycles('gpurun_out/tr5_${DT:-f64}_p0.bin')
" > gpurun_out/tr5_wa.txt 2>&1
rm -f gpurun_out/tr5_*.bin
