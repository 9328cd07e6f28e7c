# A/B: run bench.py (c3, kernel timing) with each library variant named on the command line.
# usage: bash tools/gpu/ab.sh base pc1 pc4 ...   ("base" = the in-tree build)
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
CFG=${CFG:-c3}
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so; else cp tools/liboomb_$v.so paper_2602_02108_b200/liboomb.so; fi
  timeout 900 python bench.py --config $CFG --steps ${STEPS:-2} --warmup 3 --no-cpu --no-e2e --offload-cap 0 > gpurun_out/ab_${v}_$rep.json 2> gpurun_out/ab_${v}_$rep.err
  python - "$v" "$rep" <<'PY'
import json, sys
v, rep = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}_{rep}.json").read().strip().splitlines()[-1])
    k = d.get("kernels", {})
    print(f"{v:10s} rep{rep} ms/step {d['ms_per_step']:.1f}  frac {d['roofline']['frac']:.3f}  clocks {d['clocks']['sm_mhz']}  " +
          "  ".join(f"{n}={k[n]['ms_per_step']:.1f}" for n in ("fwd_phase", "bwd_phase", "score") if n in k))
except Exception as e:
    print(v, rep, "failed", e, open(f"gpurun_out/ab_{v}_{rep}.err").read()[-800:])
PY
done
done
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
