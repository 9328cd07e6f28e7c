set -u
mkdir -p gpurun_out
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
for v in kvtrace kvtracep; do
cp tools/liboomb_$v.so paper_2602_02108_b200/liboomb.so
OOMB_CTA_TRACE=dkdv:10:gpurun_out/kv_$v.bin timeout 600 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2>&1
echo "== $v"; python tools/kv_trace.py gpurun_out/kv_$v.bin 1500
done
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
