set -x
python paper_2407_19892_b200/build.py >/dev/null 2>&1 || true
export MP_N=200000 MP_K=64
VARIANTS="mmaprof" DBGS="0" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64"
VARIANTS="mmaprof_dbg" DBGS="2 4 3" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64"
VARIANTS="epiblock_prof" DBGS="0" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64"
for i in 1 2; do
  timeout 120 python tools/sym_probe.py 2>&1 | grep "n=" | sed "s/^/[base] /" | cut -c1-120
  GGM_LIB_PATH=tools/variants/epiblock.so timeout 120 python tools/sym_probe.py 2>&1 | grep "n=" | sed "s/^/[epiblock] /" | cut -c1-120
done
