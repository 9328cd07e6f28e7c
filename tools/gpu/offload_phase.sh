set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/offload_timeline.py 2>&1 | grep -E "^== |write-backs"
