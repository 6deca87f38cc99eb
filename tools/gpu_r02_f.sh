#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
timeout 1200 python -m pytest tests/test_gpu_controller.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_f.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_f.log | tail -2; grep -E "^FAILED" gpurun_out/pytest_f.log | head
cat gpurun_out/dequant_counts.json; echo
for v in default m3; do
  lib=paper_2206_11357_b200/libgact.so; [ $v != default ] && lib=build/var_$v/libgact.so
  GACT_LIB_PATH=$lib python tools/qtime.py --dtypes bf16,f16
  for w in resnet50 bert_layer gcn_swin; do
  GACT_LIB_PATH=$lib python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['phases']['quantize_frac'], d['phases']['dequantize_frac'], d['clocks']['sm_mhz'])"
  done
done
