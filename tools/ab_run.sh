# Same-session A/B driver (GPU box): the default libggm.so against tools/variants/$V.so
# (built by tools/build_variant.sh), alternating three times.  Default: the symmetric-scheme
# stage timings at C4/C5 sizes (tools/sym_ab.py); SOLVE=1: the C3 eigenvalue-MLE kernel
# (tools/solve_ab.py; FP=<passes> for a fixed pass count).  Log: gpurun_out/ab_$V.log
set -u
mkdir -p gpurun_out
V=${V:?variant name}
S=tools/sym_ab.py
[ -n "${SOLVE:-}" ] && S=tools/solve_ab.py
for i in 1 2 3; do
  FIXED_PASSES=${FP:-} timeout 300 python $S
  FIXED_PASSES=${FP:-} GGM_LIB_PATH=tools/variants/$V.so TAG=$V timeout 300 python $S
done > gpurun_out/ab_$V.log 2>&1
cat gpurun_out/ab_$V.log
