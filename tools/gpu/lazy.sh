set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_layer_loop.py tests/test_gpu_offload.py tests/test_gpu_offload_fullsize.py tests/test_gpu_tier_attach.py tests/test_gpu_model_step.py tests/test_gpu_errors.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|^E " | head -12
export OOMB_TIER_DEBUG=1
for lz in 1 0; do echo "== lazy $lz"; OOMB_TIER_LAZY_WB=$lz timeout 900 python tools/offload_timeline.py 2>&1 | grep -E "^== capped|^h2d|forced|chunks with"; done
