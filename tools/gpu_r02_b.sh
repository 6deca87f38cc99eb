#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
for v in tma tmap prmt; do
GACT_LIB_PATH=build/var_$v/libgact.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "256 or batch or tiny or edge or c1" > gpurun_out/pytest_$v.log 2>&1
echo "$v pytest rc=$?"; tail -2 gpurun_out/pytest_$v.log
done
python tools/qtime.py --dtypes bf16
for v in tma tmap prmt; do GACT_LIB_PATH=build/var_$v/libgact.so python tools/qtime.py --dtypes bf16; done
for v in default tma tmap; do
  lib=paper_2206_11357_b200/libgact.so; [ $v != default ] && lib=build/var_$v/libgact.so
  GACT_LIB_PATH=$lib python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['phases'])"
done
