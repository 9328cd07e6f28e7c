set -u
KREGEX=attn_fwd bash tools/gpu/ab_ncu.sh base f4x2 f4x2p f4p
KREGEX=score bash tools/gpu/ab_ncu.sh base sthi
bash tools/gpu/ab.sh base f4x2p sthi
cp paper_2602_02108_b200/liboomb.so /tmp/lb.so; cp tools/liboomb_sthi.so paper_2602_02108_b200/liboomb.so
timeout 900 python -m pytest tests/test_gpu_parity.py -k "scor or select" tests/test_gpu_bench_data.py tests/test_gpu_oracle_chunks.py tests/test_gpu_fullsize.py -q -x -s -p no:cacheprovider 2>&1 | grep -i "passed\|failed\|error\|bench-data\|assert" | head -20
cp /tmp/lb.so paper_2602_02108_b200/liboomb.so
