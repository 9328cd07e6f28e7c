# A/B: copy-stream priority for the staged page moves (c3 offload key), alternating
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
for rep in 1 2; do
for v in 1 0; do
  OOMB_TIER_PRIO=$v timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/pab_${v}_$rep.json 2> gpurun_out/pab_${v}_$rep.err
  python -c "
import json; d=json.loads(open('gpurun_out/pab_${v}_$rep.json').read().strip().splitlines()[-1])['offload']
print('prio_high=$v rep $rep', 'bench', round(d['bench_data']['exposed_pct'],1), 'low', round(d['low_locality']['exposed_pct'],1), [(x['device_slots'], round(x['exposed_pct'],1)) for x in d['low_locality_slot_sweep']])"
done
done
timeout 900 python -m pytest tests/test_gpu_offload.py tests/test_gpu_layer_loop.py -q -x -p no:cacheprovider 2>&1 | tail -1
