#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
echo "parity: $(timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
for pass in 1 2; do
for d in default build/var_smallold; do
  lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
  for G in 32 64 128; do for spec in "bf16 4" "f32 4"; do set -- $spec
    echo "$pass $d $(GACT_LIB_PATH=$lib python tools/prof_kernels.py --G $G --dtype $1 --bits $2 --reps 1 2>&1 | tail -1)"
  done; done
done
done
exit 0
