#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
echo "late3 parity: $(GACT_LIB_PATH=build/var_late3/libgact.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1)"
for pass in 1 2; do
for d in default build/var_late2 build/var_late3; do
  lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
  for w in "resnet50 bf16" "bert_layer bf16"; do set -- $w
  echo "$pass $d $1 $2 $(GACT_LIB_PATH=$lib python bench.py --workload $1 --dtype $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases']['quantize_ms'])")"
  done
done
done
exit 0
