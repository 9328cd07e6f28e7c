set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KREGEX='score_' bash tools/gpu/ab_ncu.sh base scpair 2>&1 | tail -3
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
cp tools/liboomb_scpair.so paper_2602_02108_b200/liboomb.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_bench_data.py tests/test_gpu_oracle_chunks.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|^E " | head -5
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
