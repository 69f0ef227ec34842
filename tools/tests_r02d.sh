# Full GPU suite on the default and the checked (-DGGM_CHECKED) library, and smoke()
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "pytest rc=$?"
GGM_LIB_PATH=tools/variants/checked.so timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02d_pytest_gpu_checked.log 2>&1; echo "pytest checked rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc=$?"
