# Round-2 re-entry check of HEAD (one gpurun session): full GPU suite, smoke, bench lines C5 and C4.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02y_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02y_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02y_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config C4 --no-stages > gpurun_out/r02y_bench_c4.json 2> gpurun_out/r02y_bench_c4.err; echo "bench C4 rc=$?"
