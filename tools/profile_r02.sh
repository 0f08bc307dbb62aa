# Round-2 evidence on the GPU box: bench line (default contract run), ncu launch
# list of one reduction (fp64 + fp32), one ncu --set full capture each of the
# v6 (last pass) and first v5 pass kernels.  usage: tools/profile_r02.sh TAG
set -x
TAG=${1:-r02d}
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
for DT in f64 f32; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file $OUT/launches_${TAG}_$DT.csv \
      python tools/one_run.py 32768 128 $DT 32 1 > /dev/null 2>&1
  python tools/ncu_traffic.py $OUT/launches_${TAG}_$DT.csv 32768:128:$DT:32:1 > $OUT/launches_${TAG}_${DT}_summary.txt 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_v6 -c 1 -o $OUT/full_v6_$TAG \
    python tools/one_run.py 32768 128 f64 32 1 > $OUT/ncu_full_v6_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_v5 -c 1 -o $OUT/full_v5_$TAG \
    python tools/one_run.py 32768 128 f64 32 1 > $OUT/ncu_full_v5_$TAG.log 2>&1
ls -la $OUT
