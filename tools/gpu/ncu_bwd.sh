# full ncu captures (source-level) of the backward pair at a late chunk of a 512K-token c3 run
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in attn_bwd_dq_kernel attn_bwd_dkdv_kernel; do
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 10 --launch-count 1 -f -o gpurun_out/bwd_$k python bench.py --config c3 --tokens 524288 --steps 1 --warmup 1 --no-cpu --no-e2e --offload-cap 0 > /dev/null 2>&1
python tools/ncu_hot.py gpurun_out/bwd_$k.ncu-rep 30 > gpurun_out/bwd_${k}_hot.txt 2>&1
head -40 gpurun_out/bwd_${k}_hot.txt
done
ls -la gpurun_out/*.ncu-rep
