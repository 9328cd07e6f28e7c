set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layer_loop.py tests/test_gpu_bench_data.py -q -x -p no:cacheprovider 2>&1 | tail -3
for c in c1 c3 c2; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --offload-cap 0 > gpurun_out/bench_native_$c.json 2> gpurun_out/bench_native_$c.err
python tools/bsum.py gpurun_out/bench_native_$c.json | head -3
done
OOMB_NATIVE_LOOP=0 timeout 900 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > gpurun_out/bench_py_c1.json 2>&1
python tools/bsum.py gpurun_out/bench_py_c1.json | head -2
