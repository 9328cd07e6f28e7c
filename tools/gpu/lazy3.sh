set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_layer_loop.py tests/test_gpu_offload.py tests/test_gpu_offload_fullsize.py tests/test_gpu_tier_attach.py tests/test_gpu_model_step.py tests/test_gpu_errors.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed" | tail -1
OOMB_TIER_LAZY_WB=1 timeout 1500 python -m pytest tests/test_gpu_layer_loop.py tests/test_gpu_offload.py tests/test_gpu_offload_fullsize.py tests/test_gpu_tier_attach.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed" | tail -1
