# Bench lines (C5, C4) + per-rank shares (sim_ranks N = 1 2 4 8) after the prep / merge-offset changes.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sym_stress.py tests/test_gpu_distributed_sym.py tests/test_gpu_overall.py -x -q > gpurun_out/r02aa_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02aa_pytest.log
timeout 900 python bench.py > gpurun_out/r02aa_bench.json 2> gpurun_out/r02aa_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config C4 --no-stages > gpurun_out/r02aa_bench_c4.json 2> gpurun_out/r02aa_bench_c4.err; echo "bench C4 rc=$?"
timeout 900 python tools/sim_ranks.py 1 2 4 8 > gpurun_out/r02aa_simranks.log 2>&1; echo "sim rc=$?"
tail -4 gpurun_out/r02aa_simranks.log
