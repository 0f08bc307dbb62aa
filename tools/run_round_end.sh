# round-end check: timings, smoke, full -m gpu suite, default bench line, ncu launch lists
set -x
timeout 300 python tools/quick_time.py f64 f32 > gpurun_out/roundend_qt.txt 2>&1
cat gpurun_out/roundend_qt.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/roundend_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/roundend_gputest.txt 2>&1
tail -3 gpurun_out/roundend_gputest.txt
timeout 900 python bench.py > gpurun_out/roundend_bench.json 2> gpurun_out/roundend_bench.err
for DT in f64 f32; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/launches_r02g_$DT.csv \
      python tools/one_run.py 32768 128 $DT 32 1 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_v6 -c 1 -o gpurun_out/full_v6_r02g \
    python tools/one_run.py 32768 128 f64 32 1 > gpurun_out/ncu_full_v6_r02g.log 2>&1
tail -c 400 gpurun_out/roundend_bench.json
