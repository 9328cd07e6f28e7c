set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_concurrency.py tests/test_gpu_layer_loop.py tests/test_gpu_sharding.py -q -x -p no:cacheprovider > gpurun_out/scratch_tests.log 2>&1; tail -2 gpurun_out/scratch_tests.log
for r in 1 2; do timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/c1_$r.json 2> gpurun_out/c1_$r.err; python tools/bsum.py gpurun_out/c1_$r.json 2>/dev/null | head -1; done
OOMB_LOOP_HOSTPROF=1 timeout 300 python tools/host_probe_c1.py c1 2>&1 | tail -2
bash tools/gpu/r03_stage_ab.sh
