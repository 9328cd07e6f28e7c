set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_layer_loop.py -q -x -p no:cacheprovider 2>&1 | grep -E "Error|error|assert|^E " | head -20
