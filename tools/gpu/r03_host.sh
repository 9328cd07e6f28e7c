# c1 host-issue breakdown, c1 bench with the timed steps unprofiled
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
OOMB_LOOP_HOSTPROF=1 timeout 300 python tools/host_probe_c1.py c1 > gpurun_out/host_probe_c1.log 2>&1; tail -12 gpurun_out/host_probe_c1.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/c1.json 2> gpurun_out/c1.err; python tools/bsum.py gpurun_out/c1.json 2>/dev/null | head -1
