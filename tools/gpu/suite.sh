# full GPU suite + smoke (used from gpurun)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 > gpurun_out/gpu_suite_full.log; tail -15 gpurun_out/gpu_suite_full.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
