# Same-session A/B: default candidate epilogue vs the staggered one (-DGGM_EPI_STAGGER).
set -u
mkdir -p gpurun_out
GGM_LIB_PATH=tools/variants/stagger.so timeout 900 python -m pytest tests/test_gpu_sym_stress.py tests/test_gpu_sparse.py tests/test_gpu_distributed_sym.py -x -q > gpurun_out/ab_stagger_tests.log 2>&1; echo "tests rc=$?"
for i in 1 2 3; do
  timeout 300 python tools/sym_ab.py
  GGM_LIB_PATH=tools/variants/stagger.so timeout 300 python tools/sym_ab.py
done > gpurun_out/ab_stagger.log 2>&1
cat gpurun_out/ab_stagger.log
