# Round-2 end evidence (one gpurun session): full GPU suite, smoke, bench lines (C5 with
# stages, C4), launch list of the C5 step, full ncu captures of the BK2 main launch (C5 axis
# A, C4).  TAG names the files (default r02g).
set -u
mkdir -p gpurun_out
T=${TAG:-r02g}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config C4 --no-stages > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; echo "bench C4 rc=$?"
if [ -z "${SKIP_NCU:-}" ]; then
  B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
    --launch-skip 1 --launch-count 1 -o gpurun_out/${T}_bk2 $B > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
    --launch-skip 1 --launch-count 1 -o gpurun_out/${T}_bk2_c4 $B --config C4 > gpurun_out/${T}_ncu_c4.log 2>&1; echo "ncu C4 rc=$?"
fi
