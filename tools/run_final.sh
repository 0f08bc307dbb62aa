# round-end check on the GPU box: smoke, full -m gpu suite, default bench line
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_gputest.txt 2>&1
tail -5 gpurun_out/final_gputest.txt
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
tail -c 600 gpurun_out/final_bench.json
