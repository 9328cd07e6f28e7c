set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_concurrency.py tests/test_gpu_model_step.py -q -x -p no:cacheprovider 2>&1 | tail -3
CFG=c1 STEPS=5 bash tools/gpu/ab.sh base nosplit
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c1_split.json 2>&1
python tools/bsum.py gpurun_out/bench_c1_split.json
