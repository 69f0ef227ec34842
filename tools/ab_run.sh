set -u
mkdir -p gpurun_out
V=${V:-halfn}
GGM_LIB_PATH=tools/variants/$V.so timeout 120 python tools/sym_ab.py > gpurun_out/r02h_first_$V.log 2>&1; echo "first rc=$?"; cat gpurun_out/r02h_first_$V.log
GGM_LIB_PATH=tools/variants/$V.so timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sym_stress.py tests/test_gpu_distributed_sym.py tests/test_gpu_overall.py -x -q > gpurun_out/r02h_tests_$V.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02h_tests_$V.log
for i in 1 2 3; do
  timeout 300 python tools/sym_ab.py
  GGM_LIB_PATH=tools/variants/$V.so TAG=$V timeout 300 python tools/sym_ab.py
done > gpurun_out/r02h_ab_$V.log 2>&1
cat gpurun_out/r02h_ab_$V.log
