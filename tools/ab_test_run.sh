# GPU box: symmetric-scheme tests on the default build, then the A/B against variant $V.
set -u
mkdir -p gpurun_out
V=${V:?variant}
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sym_stress.py tests/test_gpu_distributed_sym.py tests/test_gpu_overall.py tests/test_gpu_configs.py tests/test_gpu_determinism.py -x -q > gpurun_out/ab_tests_default.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests_default.log
V=$V bash tools/ab_run.sh
