# Part-major unit shares (sim_ranks, default vs GGM_SYM_ASSIGN=strided, and --symB), the x64
# TMEM-load epilogue variant (A/B), new tests.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed_sym.py tests/test_gpu_sparse.py -x -q > gpurun_out/r02ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02ab_pytest.log
timeout 900 python tools/sim_ranks.py 1 2 4 8 > gpurun_out/r02ab_simranks_part.log 2>&1; echo "sim part rc=$?"
GGM_SYM_ASSIGN=strided timeout 900 python tools/sim_ranks.py 1 2 4 8 > gpurun_out/r02ab_simranks_strided.log 2>&1; echo "sim strided rc=$?"
timeout 900 python tools/sim_ranks.py 1 2 4 8 --symB > gpurun_out/r02ab_simranks_symB.log 2>&1; echo "sim symB rc=$?"
for i in 1 2 3; do
  timeout 300 python tools/sym_ab.py
  GGM_LIB_PATH=tools/variants/ld64.so timeout 300 python tools/sym_ab.py
done > gpurun_out/r02ab_ld64.log 2>&1
cat gpurun_out/r02ab_ld64.log
