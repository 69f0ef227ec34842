set -u
mkdir -p gpurun_out
V=${V:-thrshfl}
for i in 1 2 3; do
  timeout 300 python tools/sym_ab.py
  GGM_LIB_PATH=tools/variants/$V.so TAG=$V timeout 300 python tools/sym_ab.py
done > gpurun_out/r02h_ab_$V.log 2>&1
cat gpurun_out/r02h_ab_$V.log
