#!/bin/bash
cd "$(dirname "$0")/.."
make oracle >/dev/null
echo "tests: $(timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1)"
for pass in 1 2; do
for d in default build/var_g2048old; do
  lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
  for spec in "bf16 1" "bf16 4" "bf16 8" "f16 2"; do set -- $spec
    echo "$pass $d $(GACT_LIB_PATH=$lib python tools/prof_kernels.py --G 2048 --dtype $1 --bits $2 --reps 1 2>&1 | tail -1)"
  done
done
done
exit 0
