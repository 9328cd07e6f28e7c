# compute-sanitizer memcheck over the tcgen05 kernels on small parity cases
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
for t in "tests/test_gpu_parity.py::test_attention_bf16_parity" "tests/test_gpu_parity.py::test_tc_scorer_matches_exact_scorer" "tests/test_gpu_concurrency.py" "tests/test_gpu_parity.py::test_tc_forward_dense_qwen_chunk"; do
  timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 17 python -m pytest -q -x "$t" > gpurun_out/san_$(echo $t | tr '/:' '__').log 2>&1
  echo "$t rc=$?"; grep -m3 "ERROR SUMMARY\|Invalid\|passed\|failed" gpurun_out/san_$(echo $t | tr '/:' '__').log
done
