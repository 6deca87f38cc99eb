#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
GACT_LIB_PATH=build/var_xg/libgact.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "512 or 1024 or 2048 or batch or tiny" > gpurun_out/pytest_xg.log 2>&1
echo "xg pytest rc=$?"; tail -1 gpurun_out/pytest_xg.log
for G in 512 1024 2048; do
for v in default xg; do
  lib=paper_2206_11357_b200/libgact.so; [ $v != default ] && lib=build/var_$v/libgact.so
  GACT_LIB_PATH=$lib python tools/qtime.py --dtypes bf16 --G $G
done; done
