set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2602_02108_b200/liboomb.so /tmp/lb_base.so
cp tools/liboomb_kv3.so paper_2602_02108_b200/liboomb.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_concurrency.py tests/test_gpu_oracle_chunks.py tests/test_gpu_fullsize.py tests/test_gpu_layer_loop.py tests/test_gpu_sharding.py -q -x -p no:cacheprovider > gpurun_out/kv3_tests.log 2>&1
tail -3 gpurun_out/kv3_tests.log
cp /tmp/lb_base.so paper_2602_02108_b200/liboomb.so
KREGEX=attn_bwd_dkdv bash tools/gpu/ab_ncu.sh base kv3
bash tools/gpu/ab.sh base kv3
