# Per-kernel serialized durations (ncu launch list) of library variants at a 256K-token c3 run.
# usage: KREGEX='attn_bwd' bash tools/gpu/ab_ncu.sh base v1 v2 ...
set -u
mkdir -p gpurun_out
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
KREGEX=${KREGEX:-attn_}
TOK=${TOK:-262144}
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so; else cp tools/liboomb_$v.so paper_2602_02108_b200/liboomb.so; fi
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$KREGEX --csv --log-file gpurun_out/abn_$v.csv \
     python bench.py --config ${CFG:-c3} --tokens $TOK --steps 1 --warmup 1 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2> gpurun_out/abn_$v.err
  python - "$v" <<'PY'
import csv, sys, collections
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/abn_{v}.csv")) if len(r) > 10]
h = rows[0]; rows = rows[1:]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows:
    if r[mi] == "gpu__time_duration.sum":
        d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
out = []
for k, xs in sorted(d.items()):
    half = xs[len(xs) // 2:]  # the timed step (second half of the launches)
    out.append(f"{k.split('::')[-1][:22]}={sum(half)/1e6:.2f}ms/{len(half)}")
print(f"{v:8s}", "  ".join(out))
PY
done
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
