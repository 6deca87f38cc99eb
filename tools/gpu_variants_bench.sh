#!/bin/bash
# ResNet-50 bench step per tuning variant (experiments only)
cd "$(dirname "$0")/.."
for d in "" build/var_*; do
  if [ -n "$d" ]; then export GACT_LIB_PATH=$d/libgact.so; else unset GACT_LIB_PATH; fi
  python bench.py --steps 20 --warmup 3 --workload ${W:-resnet50} --dtype ${DT:-bf16} --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${d:-default}', d['value'], d['phases']['quantize_gbs'], d['phases']['dequantize_gbs'])"
done
