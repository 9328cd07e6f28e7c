set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
cp tools/liboomb_fwd5.so paper_2602_02108_b200/liboomb.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_oracle_chunks.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|^E " | head -8
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
STEPS=3 bash tools/gpu/ab.sh base fwd5 2>&1 | grep rep
