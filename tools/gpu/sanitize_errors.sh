# compute-sanitizer memcheck over the bad-page-id paths (kernels skip out-of-range ids)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 17 python -m pytest -q -x tests/test_gpu_errors.py > gpurun_out/san_errors.log 2>&1
echo "memcheck rc=$?"; grep -m3 "ERROR SUMMARY\|Invalid\|passed\|failed" gpurun_out/san_errors.log
