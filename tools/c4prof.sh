# BK2 C4 tile-time decomposition with the instrumented builds (cycles per tile on CTA 0)
export MP_N=${MP_N:-200000} MP_K=${MP_K:-64}
VARIANTS="mmaprof" DBGS="0" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64"
VARIANTS="mmaprof_dbg" DBGS="2 4 3" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64"
