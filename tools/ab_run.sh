set -u
mkdir -p gpurun_out
python -c "import __graft_entry__" 
for cfg in "200000 64" "1000000 100"; do
  set -- $cfg
  echo "#### n=$1 k=$2"
  MP_N=$1 MP_K=$2 VARIANTS="mmaprof_dbg" DBGS="2 4 3 0" bash tools/mma_prof.sh 2>&1 | grep -v "cta 64"
done > gpurun_out/r02h_mmaprof.log 2>&1
cat gpurun_out/r02h_mmaprof.log
