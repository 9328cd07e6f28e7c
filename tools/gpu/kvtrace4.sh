set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
for v in kvtrace kvtp4 kvtp2 kvtp4x2; do
cp tools/liboomb_$v.so paper_2602_02108_b200/liboomb.so
for idx in 200; do
echo "== $v chunk-launch $idx"
OOMB_CTA_TRACE=dkdv:$idx:gpurun_out/kv_$idx.bin timeout 600 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > gpurun_out/kvt_$idx.json 2> gpurun_out/kvt_$idx.err
python tools/kv_trace.py gpurun_out/kv_$idx.bin 1500
done
done
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
