set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KREGEX='attn_' bash tools/gpu/ab_ncu.sh base pairF pairKV pairKV2 pairDQ pairAll 2>&1 | tail -8
STEPS=3 bash tools/gpu/ab.sh base pairAll 2>&1 | grep rep
