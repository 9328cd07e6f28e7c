# A/B of the offload measurement (bench.py's `offload` key) between library variants, alternating
# usage: bash tools/gpu/offload_ab.sh base norestore
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so; else cp tools/liboomb_$v.so paper_2602_02108_b200/liboomb.so; fi
  timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/oab_${v}_$rep.json 2> gpurun_out/oab_${v}_$rep.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/oab_${v}_$rep.json').read().strip().splitlines()[-1])['offload']; print('$v', $rep, round(d['exposed_pct'],2), d['wall_s_capped_runs'], d['wall_s_resident_runs'])"
done
done
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
