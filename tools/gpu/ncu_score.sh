python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
for k in score_stats_kernel score_vote_kernel; do
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 200 --launch-count 1 -f -o gpurun_out/late1m_$k python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2> gpurun_out/ncu_$k.err
tail -2 gpurun_out/ncu_$k.err
done
ls -la gpurun_out/late1m_*
