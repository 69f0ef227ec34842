# GPU box: BK4 accumulator-copy count (default 8 vs 16 / 4), C3 solve kernel time.
set -u
mkdir -p gpurun_out
for i in 1 2 3; do
  TAG=g8 timeout 300 python tools/solve_ab.py
  GGM_LIB_PATH=tools/variants/red16.so TAG=g16 timeout 300 python tools/solve_ab.py
  GGM_LIB_PATH=tools/variants/red4.so TAG=g4 timeout 300 python tools/solve_ab.py
done 2>&1 | grep "C3" > gpurun_out/r02k_redgroups.log
cat gpurun_out/r02k_redgroups.log
