#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
echo "default tests: $(timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1)"
for pass in 1 2; do
for d in default build/var_qf3 build/var_fnox4m3; do
  lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
  for spec in "268435456 f32 1" "268435456 f32 4" "268435456 f32 8"; do set -- $spec
    echo "$pass $d $(GACT_LIB_PATH=$lib python tools/prof_kernels.py --n $1 --dtype $2 --bits $3 --reps 1 2>&1 | tail -1)"
  done
  for w in "resnet50 f32" "gcn f32"; do set -- $w
  echo "$pass $d $1 $2 $(GACT_LIB_PATH=$lib python bench.py --workload $1 --dtype $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases']['quantize_ms'], d['phases']['dequantize_ms'])")"
  done
done
done
exit 0
