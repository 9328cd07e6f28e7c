set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_oracle_chunks.py tests/test_gpu_layer_loop.py -q -x -p no:cacheprovider 2>&1 | tail -2
KREGEX=attn_bwd bash tools/gpu/ab_ncu.sh base nold1 kvld1
bash tools/gpu/ab.sh base nold1
cp paper_2602_02108_b200/liboomb.so /tmp/lb.so; cp tools/liboomb_kvtrace.so paper_2602_02108_b200/liboomb.so
OOMB_CTA_TRACE=dkdv:10:gpurun_out/kv_ld1.bin timeout 600 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2>&1
python tools/kv_trace.py gpurun_out/kv_ld1.bin 1500
cp /tmp/lb.so paper_2602_02108_b200/liboomb.so
