#!/bin/bash
cd "$(dirname "$0")/.."
for v in rng8 rng8p rng8q; do GACT_LIB_PATH=build/var_$v/libgact.so python tools/qtime.py --dtypes bf16; done
for v in rng8 rng8p rng8q; do
  GACT_LIB_PATH=build/var_$v/libgact.so python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['phases'])"
done
