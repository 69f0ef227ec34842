# One ncu --set full capture of the symmetric main kernel (C5 axis A) -> gpurun_out/$1.ncu-rep
set -u
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
timeout 300 $B > gpurun_out/$1_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
  --launch-skip 1 --launch-count 1 -o gpurun_out/$1 $B > gpurun_out/$1_ncu.log 2>&1; echo "ncu rc=$?"
