set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_concurrency.py tests/test_gpu_sharding.py tests/test_gpu_sharding_composed.py -q -x -p no:cacheprovider > gpurun_out/planes_tests.log 2>&1
tail -3 gpurun_out/planes_tests.log
timeout 900 python tools/offload_slack_probe.py 128 512 2048 4160 > gpurun_out/slack.log 2>&1
cat gpurun_out/slack.log | cut -c1-3000
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > gpurun_out/c4.json 2> gpurun_out/c4.err
python tools/bsum.py gpurun_out/c4.json
