#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_e.log | tail -3; grep -E "^FAILED" gpurun_out/pytest_e.log | head -20
cat gpurun_out/everygroup_counts.json gpurun_out/dequant_counts.json 2>/dev/null
for v in default m3; do
  lib=paper_2206_11357_b200/libgact.so; [ $v != default ] && lib=build/var_$v/libgact.so
  GACT_LIB_PATH=$lib python tools/qtime.py --dtypes bf16,f32
  for w in resnet50 bert_layer; do
  GACT_LIB_PATH=$lib python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['phases'])"
  done
done
