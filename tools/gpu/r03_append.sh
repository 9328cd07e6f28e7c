# staged append: parity subset, c1 + c3 bench lines
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rope.py tests/test_gpu_fuzz.py tests/test_gpu_oracle_chunks.py -q -x -p no:cacheprovider > gpurun_out/app_tests.log 2>&1; tail -2 gpurun_out/app_tests.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/c1.json 2> gpurun_out/c1.err; python tools/bsum.py gpurun_out/c1.json 2>/dev/null | head -4
timeout 900 python bench.py --no-cpu > gpurun_out/c3.json 2> gpurun_out/c3.err; python tools/bsum.py gpurun_out/c3.json 2>/dev/null | head -6
