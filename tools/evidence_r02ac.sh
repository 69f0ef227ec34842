# Folded part-major shares, x64 TMEM loads (default; ld32 = control), full GPU suite, bench lines.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ac_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02ac_pytest_gpu.log
timeout 900 python tools/sim_ranks.py 1 2 4 8 > gpurun_out/r02ac_simranks_fold.log 2>&1; echo "sim rc=$?"; tail -4 gpurun_out/r02ac_simranks_fold.log
for i in 1 2 3; do
  timeout 300 python tools/sym_ab.py
  GGM_LIB_PATH=tools/variants/ld32.so timeout 300 python tools/sym_ab.py
done > gpurun_out/r02ac_ld32.log 2>&1
cat gpurun_out/r02ac_ld32.log
timeout 900 python bench.py > gpurun_out/r02ac_bench.json 2> gpurun_out/r02ac_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config C4 --no-stages > gpurun_out/r02ac_bench_c4.json 2> gpurun_out/r02ac_bench_c4.err; echo "bench C4 rc=$?"
