#!/bin/bash
cd "$(dirname "$0")/.."
make oracle >/dev/null
echo "default parity: $(timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
echo "fsum7 parity: $(GACT_LIB_PATH=build/var_fsum7/libgact.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
for pass in 1 2; do
for d in default build/var_fsum0 build/var_fsum7; do
  lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
  for spec in "268435456 bf16 1" "268435456 bf16 2" "268435456 bf16 4" "268435456 f32 4"; do set -- $spec
    echo "$pass $d $(GACT_LIB_PATH=$lib python tools/prof_kernels.py --n $1 --dtype $2 --bits $3 --reps 1 2>&1 | tail -1)"
  done
  echo "$pass $d resnet50 $(GACT_LIB_PATH=$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases']['quantize_ms'])")"
done
done
exit 0
