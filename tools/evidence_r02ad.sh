# Pool without up-front fill (closed reservations), seed-share split of the needed rows only;
# GPU suite, A/B timing, per-rank shares, stand-alone grid pass.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ad_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02ad_pytest_gpu.log
for i in 1 2; do timeout 300 python tools/sym_ab.py; done > gpurun_out/r02ad_symab.log 2>&1; cat gpurun_out/r02ad_symab.log
timeout 900 python tools/sim_ranks.py 1 2 4 8 > gpurun_out/r02ad_simranks.log 2>&1; echo "sim rc=$?"; tail -4 gpurun_out/r02ad_simranks.log
timeout 300 python tools/solve_probe.py --pass > gpurun_out/r02ad_solve_pass.log 2>&1; cat gpurun_out/r02ad_solve_pass.log
