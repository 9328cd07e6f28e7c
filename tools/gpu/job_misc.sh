set -u
mkdir -p gpurun_out
./tools/ubench/mufu_rate > gpurun_out/mufu_rate.txt 2>&1; cat gpurun_out/mufu_rate.txt
timeout 900 python -m pytest tests/test_gpu_bench_data.py -q -x -s -p no:cacheprovider > gpurun_out/bench_data_test.log 2>&1
tail -5 gpurun_out/bench_data_test.log
