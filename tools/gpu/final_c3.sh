set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; python tools/bsum.py gpurun_out/final_c3.json 2>/dev/null | head -1
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err; python tools/bsum.py gpurun_out/final_c1.json 2>/dev/null | head -1
