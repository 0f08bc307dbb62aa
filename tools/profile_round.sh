#!/bin/bash
# Round evidence on the GPU box: bench line, ncu launch list, one ncu --set full
# capture of the first v4 pass kernel (the dominant kernel).
# usage: tools/profile_round.sh TAG [N B DTYPE TW]
set -x
TAG=${1:-r01}
N=${2:-32768}; B=${3:-128}; DT=${4:-f64}; TW=${5:-32}
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt
timeout 900 python bench.py --dtype $DT --tw $TW > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
# launch list of one reduction (cold-cache, serialised): compare shares
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python tools/one_run.py $N $B $DT $TW 1 > /dev/null 2>&1
# one full capture of the first pass kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_v4 -c 1 -o $OUT/full_$TAG \
    python tools/one_run.py $N $B $DT $TW 1 > $OUT/ncu_full_$TAG.log 2>&1
ls -la $OUT
