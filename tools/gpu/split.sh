python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "scorer or scoring" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_sharding.py -q -x 2>&1 | tail -2
CFG=c4 STEPS=1 bash tools/gpu/ab.sh base nosplit
