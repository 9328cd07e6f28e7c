# exact final tree: full GPU suite, smoke, default bench line
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r03_gpu_suite_final.log 2>&1; tail -2 gpurun_out/r03_gpu_suite_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r03_bench_c3_final.json 2> gpurun_out/r03_bench_c3_final.err; python tools/bsum.py gpurun_out/r03_bench_c3_final.json 2>/dev/null | head -1
