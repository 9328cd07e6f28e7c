# staged page moves + one host block per page; hoisted head-dim branches: offload tests, c3 bench, c1 host probe
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1200 python -m pytest tests/test_gpu_offload.py tests/test_gpu_offload_fullsize.py tests/test_gpu_layer_loop.py tests/test_gpu_model_step.py tests/test_gpu_tier_attach.py -q -x -p no:cacheprovider > gpurun_out/offload_tests.log 2>&1; tail -2 gpurun_out/offload_tests.log
timeout 300 python tools/host_probe_c1.py c1 > gpurun_out/host_probe_c1.log 2>&1; tail -5 gpurun_out/host_probe_c1.log
timeout 900 python bench.py --no-cpu > gpurun_out/c3.json 2> gpurun_out/c3.err; python tools/bsum.py gpurun_out/c3.json 2>/dev/null | head -1
