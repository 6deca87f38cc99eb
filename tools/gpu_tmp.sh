#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
echo "xs parity: $(GACT_LIB_PATH=build/var_xs/libgact.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
for pass in 1 2; do
for d in default build/var_xs; do
  lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
  for spec in "268435456 bf16 1" "268435456 bf16 2" "268435456 bf16 4" "268435456 bf16 8" "268435456 f16 4" "268435456 f32 4"; do set -- $spec
    echo "$pass $d $(GACT_LIB_PATH=$lib python tools/prof_kernels.py --n $1 --dtype $2 --bits $3 --reps 1 2>&1 | tail -1)"
  done
done
done
exit 0
