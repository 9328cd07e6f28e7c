python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for rep in 1 2; do for pr in 0 1; do
OOMB_SEL_PRIORITY=$pr timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --no-e2e --offload-cap 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prio=$pr', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
done; done
timeout 900 python tools/offload_probe2.py
