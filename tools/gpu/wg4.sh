set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2602_02108_b200/liboomb.so /tmp/liboomb_base.so
for c in c3 c1; do python tools/variant_bitwise.py save /tmp/ref_$c.pt $c; done
for v in wg4 wg4p; do
  cp tools/liboomb_$v.so paper_2602_02108_b200/liboomb.so
  for c in c3 c1; do echo "$v $c: $(timeout 300 python tools/variant_bitwise.py compare /tmp/ref_$c.pt $c 2>&1 | tail -1)"; done
done
cp tools/liboomb_wg4.so paper_2602_02108_b200/liboomb.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_readback.py tests/test_gpu_oracle_chunks.py tests/test_gpu_layer_loop.py -q -x -p no:cacheprovider 2>&1 | tail -2
cp /tmp/liboomb_base.so paper_2602_02108_b200/liboomb.so
STEPS=3 bash tools/gpu/ab.sh base wg4 wg4p 2>&1 | grep rep
