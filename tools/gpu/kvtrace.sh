set -u
mkdir -p gpurun_out
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
cp tools/liboomb_kvtrace.so paper_2602_02108_b200/liboomb.so
for idx in 10 128 230; do
OOMB_CTA_TRACE=dkdv:$idx:gpurun_out/kv_$idx.bin timeout 600 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > gpurun_out/kvt_$idx.json 2> gpurun_out/kvt_$idx.err
python tools/kv_trace.py gpurun_out/kv_$idx.bin 1500
done
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
