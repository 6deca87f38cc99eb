#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
for v in default f4; do
  lib=paper_2206_11357_b200/libgact.so; [ $v != default ] && lib=build/var_$v/libgact.so
  GACT_LIB_PATH=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py -m gpu -q -x -p no:cacheprovider -k "batch or staged or 256" > gpurun_out/pytest_k_$v.log 2>&1
  echo "$v pytest rc=$?"; tail -1 gpurun_out/pytest_k_$v.log
done
for v in default f4 f2; do
  lib=paper_2206_11357_b200/libgact.so; [ $v != default ] && lib=build/var_$v/libgact.so
  GACT_LIB_PATH=$lib python tools/qtime.py --dtypes bf16 --n 134217728
  for w in resnet50 bert_layer gcn_swin; do
  GACT_LIB_PATH=$lib python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['phases']['quantize_frac'], d['phases']['dequantize_frac'])"
  done
  for b in 1 4; do
  GACT_LIB_PATH=$lib python bench.py --workload buf256 --avg-bits $b --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v buf256 b=$b', d['value'], d['phases']['quantize_frac'], d['phases']['dequantize_frac'])"
  done
done
