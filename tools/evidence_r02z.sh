# Prep-kernel rewrite check: GPU suite subset + launch list of the C5 step.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02z_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02z_pytest_gpu.log
timeout 300 python tools/sym_ab.py
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02z_launches.csv $B > gpurun_out/r02z_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
