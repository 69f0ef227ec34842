set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sym_stress.py tests/test_gpu_configs.py tests/test_gpu_distributed_sym.py -x -q > gpurun_out/r02af_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02af_pytest.log
for i in 1 2 3; do
  timeout 300 python tools/sym_ab.py
  GGM_LIB_PATH=tools/variants/vote2.so TAG=per_chunk_vote timeout 300 python tools/sym_ab.py
done > gpurun_out/r02af_vote.log 2>&1
cat gpurun_out/r02af_vote.log
