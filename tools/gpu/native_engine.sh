# native loop with an attached TieredEngine: bitwise vs the host loop, then the bench's offload regimes
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layer_loop.py tests/test_gpu_tier_attach.py tests/test_gpu_offload.py tests/test_gpu_offload_fullsize.py tests/test_gpu_model_step.py tests/test_gpu_errors.py -q -x -p no:cacheprovider > gpurun_out/native_engine_tests.log 2>&1
tail -5 gpurun_out/native_engine_tests.log
timeout 1800 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_offload.json 2> gpurun_out/bench_offload.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_offload.json").read().strip().splitlines()[-1])
o = d["offload"]
print(json.dumps({k: v for k, v in o.items() if k not in ("bench_data", "low_locality", "note")}))
for r in ("bench_data", "low_locality", "low_locality_slot_sweep"):
    x = o.get(r)
    if x: print(r, json.dumps(x))
print("value", d["value"], "e2e", d["e2e"]["value"])
PY
tail -3 gpurun_out/bench_offload.err
