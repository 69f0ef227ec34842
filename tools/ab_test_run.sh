# GPU box: symmetric-scheme test files on the default build, then A/B against variants VARS.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sym_stress.py tests/test_gpu_distributed_sym.py tests/test_gpu_overall.py tests/test_gpu_configs.py tests/test_gpu_determinism.py -x -q > gpurun_out/ab_tests_default.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests_default.log
for v in ${VARS:-}; do V=$v bash tools/ab_run.sh; done
