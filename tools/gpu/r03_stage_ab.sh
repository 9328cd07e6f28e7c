# A/B of staged page moves per direction (OOMB_TIER_STAGED bit 0 H2D, bit 1 D2H), c3 offload key, alternating
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
for rep in 1; do
for v in 3 1 2; do
  OOMB_TIER_STAGED=$v timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/sab_${v}_$rep.json 2> gpurun_out/sab_${v}_$rep.err
  python -c "
import json; d=json.loads(open('gpurun_out/sab_${v}_$rep.json').read().strip().splitlines()[-1])['offload']
print('staged=$v rep $rep', 'bench', round(d['bench_data']['exposed_pct'],1), 'low', round(d['low_locality']['exposed_pct'],1), [(x['device_slots'], round(x['exposed_pct'],1)) for x in d['low_locality_slot_sweep']])"
done
done
