# round-2 bench lines of every BASELINE config (builder runs; the driver re-runs c3)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; python tools/bsum.py gpurun_out/final_c3.json 2>/dev/null | head -1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref_c3.json 2> gpurun_out/final_ref_c3.err; tail -c 400 gpurun_out/final_ref_c3.json
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; python tools/bsum.py gpurun_out/final_c2.json 2>/dev/null | head -1
timeout 1500 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; python tools/bsum.py gpurun_out/final_c4.json 2>/dev/null | head -1
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err; python tools/bsum.py gpurun_out/final_c5.json 2>/dev/null | head -1
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err; python tools/bsum.py gpurun_out/final_c1.json 2>/dev/null | head -1
