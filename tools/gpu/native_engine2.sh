set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layer_loop.py tests/test_gpu_tier_attach.py tests/test_gpu_offload.py tests/test_gpu_offload_fullsize.py tests/test_gpu_bench.py -q -x -p no:cacheprovider > gpurun_out/native_engine_tests.log 2>&1
tail -5 gpurun_out/native_engine_tests.log
