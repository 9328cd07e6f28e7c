# A/B over an environment variable: bash tools/gpu/envab.sh VAR v1 v2 ...
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
VAR=$1; shift
for rep in 1 2; do for val in "$@"; do
env $VAR=$val timeout 900 python bench.py --config ${CFG:-c3} --steps ${STEPS:-2} --warmup 3 --no-cpu --no-e2e --offload-cap 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d.get('kernels',{})
print('$VAR=$val', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], '  '.join(f'{n}={k[n][\"ms_per_step\"]:.1f}' for n in ('attn_fwd','bwd_pair') if n in k))"
done; done
