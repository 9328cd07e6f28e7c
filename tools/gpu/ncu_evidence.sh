python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
# launch list of the bench command (1 timed step at full c3 size)
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_1m.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2> gpurun_out/launches_c3_1m.err
tail -1 gpurun_out/launches_c3_1m.err
# full capture of the forward kernel at a late chunk of the 1M run
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_tc4_kernel --launch-skip 200 --launch-count 1 -f -o gpurun_out/late1m_fwd4 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2>&1
for k in attn_bwd_dq_kernel attn_bwd_dkdv_kernel; do
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 200 --launch-count 1 -f -o gpurun_out/late1m_$k python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2>&1
done
ls -la gpurun_out/late1m_* gpurun_out/launches_c3_1m.csv
