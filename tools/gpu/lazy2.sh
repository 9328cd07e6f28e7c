set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export OOMB_TIER_DEBUG=1
for cfg in "0 256" "1 256" "1 512" "1 768"; do set -- $cfg; echo "== slots 7168 lazy $1 window $2"; OOMB_TIER_LAZY_WB=$1 OOMB_TIER_CLEAN_AHEAD=$2 timeout 900 python tools/offload_timeline.py --slots 7168 2>&1 | grep -E "^== |forced" | tail -3; done
for cfg in "1 128" "1 384"; do set -- $cfg; echo "== slots 6656 lazy $1 window $2"; OOMB_TIER_LAZY_WB=$1 OOMB_TIER_CLEAN_AHEAD=$2 timeout 900 python tools/offload_timeline.py 2>&1 | grep -E "^== |forced" | tail -3; done
