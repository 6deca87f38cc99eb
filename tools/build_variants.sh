#!/bin/bash
# Build tuning variants of libgact.so into build/var_<name>/ (experiments only).
# Usage: tools/build_variants.sh "name:-DGACT_Q_UNIT=4 -DGACT_Q_MINB=2" ...
cd "$(dirname "$0")/.."
NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-ffp-contract=off -Iinclude"
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  d=build/var_$name; mkdir -p $d
  for f in paper_2206_11357_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    /usr/local/cuda/bin/nvcc $NVFLAGS $defs -Xptxas -v -c -o $d/$b.o $f 2> $d/$b.log &
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/libgact.so $d/*.o
  echo "$name: $(grep -A2 'quantize_big_kernelILi1ELi4ELi1ELi1ELb0' $d/gact_quantize.log | grep -o 'Used [0-9]* registers') | dq: $(grep -A2 'dequantize_kernelILi1ELi4ELi1E' $d/gact_dequant.log | grep -o 'Used [0-9]* registers')"
done
