set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_readback.py tests/test_gpu_layer_loop.py tests/test_gpu_concurrency.py tests/test_gpu_parity.py tests/test_gpu_oracle_chunks.py -q -x -p no:cacheprovider 2>&1 | grep -E "^E |Error|assert" | head -20
for c in c1 c3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --offload-cap 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'])"; done
