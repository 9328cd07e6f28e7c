set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KREGEX='attn_fwd' bash tools/gpu/ab_ncu.sh base fwd5 fwd5p fwd4p 2>&1 | tail -6
