python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
t="tests/test_gpu_parity.py::test_attention_bf16_parity"
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -q -x "$t" > gpurun_out/san_sync.log 2>&1; echo "synccheck rc=$?"; grep -m3 "ERROR SUMMARY\|passed\|failed" gpurun_out/san_sync.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_offload.py tests/test_gpu_model_step.py tests/test_gpu_sharding.py > gpurun_out/san_mem2.log 2>&1; echo "memcheck offload/model/sharding rc=$?"; grep -m3 "ERROR SUMMARY\|passed\|failed" gpurun_out/san_mem2.log
