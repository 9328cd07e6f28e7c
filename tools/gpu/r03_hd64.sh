# head-dim-64 MMA trimming (K = hd steps, N = hd descriptors): parity, c1 bench + launch list, c3 bench
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_suite_full.log 2>&1; tail -2 gpurun_out/gpu_suite_full.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/c1.json 2> gpurun_out/c1.err; python tools/bsum.py gpurun_out/c1.json 2>/dev/null | head -4
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file gpurun_out/c1_launches.csv python bench.py --config c1 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/c1_ncu.log 2>&1; echo ncu rc $?
timeout 900 python bench.py --no-cpu > gpurun_out/c3.json 2> gpurun_out/c3.err; python tools/bsum.py gpurun_out/c3.json 2>/dev/null | head -6
