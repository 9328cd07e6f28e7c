# compute-sanitizer over the final kernels: racecheck on the backward (fused prep/schedule kernel,
# read-back epilogue, packed FMA-pipe exponentials) and memcheck on the native loop with the engine
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
run() {  # tool, test
  local log=gpurun_out/san2_$1_$(echo $2 | tr '/:[]' '____').log
  timeout 1800 compute-sanitizer --tool $1 --print-limit 20 --error-exitcode 17 python -m pytest -q -x -p no:cacheprovider "$2" > $log 2>&1
  echo "## $1 $2 rc=$?"; grep -m3 "ERROR SUMMARY\|RACECHECK SUMMARY\|Invalid\|hazard\|passed\|failed" $log
}
run racecheck "tests/test_gpu_readback.py"
run racecheck "tests/test_gpu_parity.py::test_attention_bf16_parity"
run memcheck "tests/test_gpu_readback.py"
run memcheck "tests/test_gpu_concurrency.py"
run memcheck "tests/test_gpu_offload.py"
