set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/final_c1.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("gpu_launches"))
for k, v in d.get("kernels", {}).items():
    print(k, {a: b for a, b in v.items() if a != "note"})
PY
