# GPU box: symmetric-scheme tests on variant $V, then the A/B against the default build.
set -u
mkdir -p gpurun_out
V=${V:?variant}
GGM_LIB_PATH=tools/variants/$V.so timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sym_stress.py tests/test_gpu_distributed_sym.py -x -q > gpurun_out/ab_tests_$V.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests_$V.log
V=$V bash tools/ab_run.sh
