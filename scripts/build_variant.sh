#!/bin/bash
# Build a variant of the product library with extra nvcc defines for an A/B
# run on the GPU box: scripts/build_variant.sh NAME "-DFOO=1 ..." -> build/var_NAME.so
# (scripts/ab_lib.sh swaps it in place of paper_2305_02522_b200/libbitgnn_b200.so).
set -e
name=$1; extra=$2
d=build/var_$name; mkdir -p $d
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O3 -std=c++17 $ARCH -lineinfo -Iinclude -Xcompiler -fPIC --expt-relaxed-constexpr $extra"
objs=""
for f in paper_2305_02522_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  if [ -n "$3" ] && ! echo " $3 " | grep -q " $b "; then objs="$objs build/$b.o"; continue; fi
  $NVCC $FLAGS -Xptxas -v -c -o $d/$b.o $f 2> $d/$b.ptxas.log &
  objs="$objs $d/$b.o"
done
wait
$NVCC $ARCH -shared -cudart static -Xlinker --version-script=paper_2305_02522_b200/csrc/exports.map -o build/var_$name.so $objs -ldl
echo built build/var_$name.so
