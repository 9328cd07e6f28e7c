# round-2 ncu evidence: launch list of the c3 bench step + --set full captures of the hot kernels
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3_1m.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2> gpurun_out/r02_launches.err
tail -2 gpurun_out/r02_launches.err
cap() {  # kernel, launch-skip
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$1 --launch-skip $2 --launch-count 1 -f -o gpurun_out/r02_$1 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2>&1
}
cap attn_fwd_tc4_kernel 200
cap attn_bwd_dq_kernel 40
cap attn_bwd_dkdv_kernel 40
cap score_stats_kernel 200
cap score_vote_kernel 200
ls -la gpurun_out/r02_*
python tools/ncu_traffic.py gpurun_out/r02_ncu_traffic.json "ncu --set full --clock-control none, c3 at 1M context: forward / scorer launch 201 (chunk 200, 6,400 candidate pages), backward launch 41 (chunk 215, 6,880 candidate pages), 64 selected per query page" attn_fwd_tc4=gpurun_out/r02_attn_fwd_tc4_kernel.ncu-rep attn_bwd_dq=gpurun_out/r02_attn_bwd_dq_kernel.ncu-rep attn_bwd_dkdv=gpurun_out/r02_attn_bwd_dkdv_kernel.ncu-rep score_stats=gpurun_out/r02_score_stats_kernel.ncu-rep score_vote=gpurun_out/r02_score_vote_kernel.ncu-rep
