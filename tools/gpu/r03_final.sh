# round-3 final evidence: full GPU suite + smoke, bench lines c1-c5 + reference arm, c3 launch list,
# ncu --set full of the staged append at c3
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r03_gpu_suite.log 2>&1; tail -2 gpurun_out/r03_gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r03_smoke.log 2>&1; tail -1 gpurun_out/r03_smoke.log
timeout 900 python bench.py > gpurun_out/r03_bench_c3.json 2> gpurun_out/r03_bench_c3.err; python tools/bsum.py gpurun_out/r03_bench_c3.json 2>/dev/null | head -1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r03_bench_reference_arm.json 2> gpurun_out/r03_ref.err; tail -c 300 gpurun_out/r03_bench_reference_arm.json
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/r03_bench_c1.json 2> gpurun_out/r03_c1.err; python tools/bsum.py gpurun_out/r03_bench_c1.json 2>/dev/null | head -1
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/r03_bench_c2.json 2> gpurun_out/r03_c2.err; python tools/bsum.py gpurun_out/r03_bench_c2.json 2>/dev/null | head -1
timeout 1500 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r03_bench_c4.json 2> gpurun_out/r03_c4.err; python tools/bsum.py gpurun_out/r03_bench_c4.json 2>/dev/null | head -1
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/r03_bench_c5.json 2> gpurun_out/r03_c5.err; python tools/bsum.py gpurun_out/r03_bench_c5.json 2>/dev/null | head -1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file gpurun_out/r03_launches_c3_1m.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > gpurun_out/r03_ncu_list.log 2>&1; echo ncu list rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:append_staged --launch-skip 200 --launch-count 1 \
  -o gpurun_out/r03_append_c3 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > gpurun_out/r03_ncu_append.log 2>&1; echo ncu append rc $?
