# Round-1 (j) evidence: full GPU suite and launch list of the final build (kernels of BK2
# unchanged since r01i; spectrum / solve changed).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01j_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r01j_pytest_gpu.log
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r01j_launches.csv $B > gpurun_out/r01j_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
