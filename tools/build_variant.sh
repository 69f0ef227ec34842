#!/bin/bash
# Build libggm.so with extra nvcc defines into tools/variants/<name>.so (for same-session A/B).
# Usage: tools/build_variant.sh NAME -DFOO=1 ...
set -e
name=$1; shift
d=$(mktemp -d)
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2407_19892_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $*"
for f in ggm_api sparse_precision grid_solve gram_eig gram_tc wald; do nvcc $F -c $C/$f.cu -o $d/$f.o & done; wait
mkdir -p $R/tools/variants
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/variants/$name.so $d/*.o -lcublas -lcusolver -lcusparse -L/usr/local/cuda/lib64 -Xlinker -rpath,/usr/local/cuda/lib64
rm -rf $d; echo built tools/variants/$name.so
