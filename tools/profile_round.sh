#!/bin/bash
# Round evidence on the GPU box: bench line, ncu launch list, one ncu --set full capture.
# usage: tools/profile_round.sh TAG [extra bench args]
set -x
TAG=${1:-r01}; shift
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt
timeout 900 python bench.py "$@" > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
# launch list of one reduction (cold-cache, serialised): compare shares
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python tools/one_run.py 32768 128 f64 16 1 > /dev/null 2>&1
# one full capture of the first pass kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_ -c 1 -o $OUT/full_$TAG \
    python tools/one_run.py 32768 128 f64 16 1 > $OUT/ncu_full_$TAG.log 2>&1
ls -la $OUT
