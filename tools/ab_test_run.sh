# GPU box: distributed-scheme tests, then the per-rank shares (sim_ranks N = 1 2 4 8).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed_sym.py tests/test_gpu_sparse.py tests/test_gpu_overall.py -x -q > gpurun_out/r02k_pytest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02k_pytest.log
timeout 800 python tools/sim_ranks.py 1 2 4 8 > gpurun_out/r02k_simranks.log 2>&1; echo "sim rc=$?"; tail -4 gpurun_out/r02k_simranks.log
