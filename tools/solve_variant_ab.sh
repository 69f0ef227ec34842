# Same-session A/B of BK4 library variants (tools/build_variant.sh NAME -D...): C3 solve
# kernel time and fixed-pass time per variant, twice.  Usage: VARIANTS="tree" bash tools/solve_variant_ab.sh
set -u
mkdir -p gpurun_out
L=gpurun_out/${TAG:-solve}_ab.log
for i in 1 2; do
  TAG=base python tools/solve_ab.py >> $L 2>&1
  TAG=base FIXED_PASSES=2000 python tools/solve_ab.py >> $L 2>&1
  for v in $VARIANTS; do
    TAG=$v GGM_LIB_PATH=tools/variants/$v.so python tools/solve_ab.py >> $L 2>&1
    TAG=$v FIXED_PASSES=2000 GGM_LIB_PATH=tools/variants/$v.so python tools/solve_ab.py >> $L 2>&1
  done
done
cat $L
