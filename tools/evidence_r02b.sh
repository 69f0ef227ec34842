# Round-2 final-build evidence (one gpurun session): bench lines (C5 default, C4), launch list of the C5
# step, full captures of BK2 (C5 axis A main launch and C4 main launch), BK4 (C3 solve) and
# the tensor-core Gram (one PBMC-scale chunk launch).  Part 1 of 2 (the session copies
# back at most 64 MiB of gpurun_out/): bench lines, launch list, BK2 captures.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02b_smi.txt
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config C4 --no-stages > gpurun_out/r02b_bench_c4.json 2> gpurun_out/r02b_bench_c4.err; echo "bench C4 rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02b_launches.csv $B > gpurun_out/r02b_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
  --launch-skip 1 --launch-count 1 -o gpurun_out/r02b_bk2 $B > gpurun_out/r02b_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
  --launch-skip 1 --launch-count 1 -o gpurun_out/r02b_bk2_c4 $B --config C4 > gpurun_out/r02b_ncu_c4.log 2>&1; echo "ncu C4 rc=$?"
