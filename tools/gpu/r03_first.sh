# re-entry check: build, c1 bench + launch list, full GPU suite + smoke
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/c1.json 2> gpurun_out/c1.err; python tools/bsum.py gpurun_out/c1.json 2>/dev/null | head -3
OOMB_NO_CLOCKS=1 timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
  --log-file gpurun_out/c1_launches.csv python bench.py --config c1 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/c1_ncu.log 2>&1; echo ncu rc $?
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_suite_full.log 2>&1; tail -3 gpurun_out/gpu_suite_full.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
