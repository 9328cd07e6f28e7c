set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/r03_bench_c1_e2e.json 2> gpurun_out/r03_c1_e2e.err; python tools/bsum.py gpurun_out/r03_bench_c1_e2e.json 2>/dev/null | head -1; tail -3 gpurun_out/r03_c1_e2e.err
