# Round-1 (k) evidence: bench line + launch list + BK2 full capture of the final build
# (lean hi-only MMA issue loop).
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r01k_bench.json 2> gpurun_out/r01k_bench.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r01k_launches.csv $B > gpurun_out/r01k_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
  --launch-skip 1 --launch-count 1 -o gpurun_out/r01k_bk2 $B > gpurun_out/r01k_ncu_full.log 2>&1; echo "ncu full rc=$?"
