# Round-2 final-build evidence (one gpurun session): bench lines (C5 default, C4), launch list of the C5
# step, full captures of BK2 (C5 axis A main launch and C4 main launch), BK4 (C3 solve) and
# the tensor-core Gram (one PBMC-scale chunk launch).  Part 2 of 2: BK4, Gram, row-mass
# captures and the overall-rules phase timing.
set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 \
  -o gpurun_out/r02b_bk4 python tools/solve_probe.py --ncu > gpurun_out/r02b_ncu_bk4.log 2>&1; echo "ncu bk4 rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:gram_tc_kernel -c 1 \
  -o gpurun_out/r02b_gramtc python tools/pbmc_probe.py > gpurun_out/r02b_ncu_gramtc.log 2>&1; echo "ncu gram_tc rc=$?"
timeout 900 bash tools/ncu_mass.sh r02b_mass > gpurun_out/r02b_ncu_mass.log 2>&1; echo "ncu mass rc=$?"
timeout 600 python tools/overall_one.py > gpurun_out/r02b_overall.log 2>&1; echo "overall rc=$?"
