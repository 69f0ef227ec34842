# Round-1 (i) evidence: full GPU suite, bench line, launch list, full ncu capture of BK2 main.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01i_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r01i_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r01i_bench.json 2> gpurun_out/r01i_bench.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
timeout 600 $B > gpurun_out/r01i_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r01i_launches.csv $B > gpurun_out/r01i_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
  --launch-skip 1 --launch-count 1 -o gpurun_out/r01i_bk2 $B > gpurun_out/r01i_ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out | tail -12
