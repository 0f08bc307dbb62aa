# v6 ring-latency probes at group sizes GS (tools/trace6.py ring())
set -x
for G in ${GS:-4 3}; do
  BB_TRACE_RING=1 BB_V6_G=$G timeout 200 python tools/trace_run6.py 32768 128 ${DT:-f64} 32 3 >> gpurun_out/tr6run.txt 2>&1
  mv gpurun_out/tr6_${DT:-f64}_n32768.bin gpurun_out/tr6_G$G.bin
  python -c "
import sys; sys.path.insert(0,'tools'); import trace6
trace6.ring('gpurun_out/tr6_G$G.bin', k=2048)
trace6.ring('gpurun_out/tr6_G$G.bin', k=20)
trace6.crossgroup('gpurun_out/tr6_G$G.bin', k=2048)
" > gpurun_out/tr6_ring_G$G.txt 2>&1
done
rm -f gpurun_out/tr6_*.bin
