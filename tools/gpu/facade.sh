set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_cpp_facade.py -q -m gpu -s 2>&1 | tail -30
