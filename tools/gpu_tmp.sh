#!/bin/bash
cd "$(dirname "$0")/.."
for pass in 1 2; do
for d in default build/var_*; do
  lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
  for spec in "134217728 bf16 2" "134217728 bf16 8" "268435456 bf16 4" "134217728 f32 4" "268435456 f32 2"; do set -- $spec
    echo "$pass $d $(GACT_LIB_PATH=$lib python tools/prof_kernels.py --n $1 --dtype $2 --bits $3 --reps 1 2>&1 | tail -1)"
  done
  [ $pass = 1 ] && echo "$d resnet50 $(GACT_LIB_PATH=$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases'])")"
done
done
