# memcheck over the session's new kernels: staged append, hd 64 tcgen05 paths, staged page moves
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x -p no:cacheprovider \
  "tests/test_gpu_parity.py::test_append_gather_kavg_bit_exact" "tests/test_gpu_parity.py::test_tc_c1_multichunk_matches_simt" \
  "tests/test_gpu_parity.py::test_tc_small_shapes_bf16_parity" > gpurun_out/r03_san_mem_kernels.log 2>&1; echo "memcheck append/hd64 rc=$?"; grep -m3 "ERROR SUMMARY\|passed\|failed" gpurun_out/r03_san_mem_kernels.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_offload.py > gpurun_out/r03_san_mem_offload.log 2>&1; echo "memcheck offload rc=$?"; grep -m3 "ERROR SUMMARY\|passed\|failed" gpurun_out/r03_san_mem_offload.log
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -q -x -p no:cacheprovider "tests/test_gpu_parity.py::test_append_gather_kavg_bit_exact" > gpurun_out/r03_san_race_append.log 2>&1; echo "racecheck append rc=$?"; grep -m3 "RACECHECK SUMMARY\|ERROR SUMMARY\|passed\|failed" gpurun_out/r03_san_race_append.log
