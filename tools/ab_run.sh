set -u
mkdir -p gpurun_out
V=${V:-ilp4}
for i in 1 2 3; do
  FIXED_PASSES=${FP:-} timeout 300 python tools/solve_ab.py
  FIXED_PASSES=${FP:-} GGM_LIB_PATH=tools/variants/$V.so TAG=$V timeout 300 python tools/solve_ab.py
done > gpurun_out/r02i_ab_$V.log 2>&1
cat gpurun_out/r02i_ab_$V.log
