VARIANTS="mmaprof_dbg" DBGS="2 3 0" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64" | grep -v EPIPROF
VARIANTS="nw2" DBGS="1" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64" | grep -v EPIPROF
