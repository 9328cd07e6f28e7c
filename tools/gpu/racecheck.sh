# compute-sanitizer racecheck (shared-memory hazards) over the tcgen05 kernels and the SIMT paths on
# small parity cases, plus memcheck over the round-2 additions (hd 64 / P 64 tcgen05, composed sharding)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
run() {  # tool, test
  local log=gpurun_out/san_$1_$(echo $2 | tr '/:[]' '____').log
  timeout 1800 compute-sanitizer --tool $1 --print-limit 20 --error-exitcode 17 python -m pytest -q -x -p no:cacheprovider "$2" > $log 2>&1
  echo "## $1 $2 rc=$?"; grep -m3 "ERROR SUMMARY\|RACECHECK SUMMARY\|Invalid\|hazard\|passed\|failed" $log
}
run racecheck "tests/test_gpu_parity.py::test_attention_bf16_parity"
run racecheck "tests/test_gpu_parity.py::test_tc_scorer_matches_exact_scorer"
run racecheck "tests/test_gpu_parity.py::test_tc_forward_dense_qwen_chunk"
run racecheck "tests/test_gpu_fuzz.py"
run memcheck "tests/test_gpu_parity.py::test_tc_small_shapes_bf16_parity"
run memcheck "tests/test_gpu_parity.py::test_tc_c1_multichunk_matches_simt"
run memcheck "tests/test_gpu_sharding_composed.py"
