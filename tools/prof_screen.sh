set -u
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/screen_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/screen_pytest.log
timeout 300 python bench.py --no-stages --no-cpu > gpurun_out/bench_screen3.json 2>gpurun_out/bench_screen3.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-stages"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_recon_topk \
  --launch-skip 1 --launch-count 1 -o gpurun_out/screen_bk2 $B > gpurun_out/screen_ncu.log 2>&1; echo "ncu rc=$?"
