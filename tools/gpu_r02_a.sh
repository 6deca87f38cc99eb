#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -m gpu -q -x -p no:cacheprovider -k "batch or bench or nccl" > gpurun_out/pytest_a.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_a.log
python tools/qtime.py --dtypes bf16,f16
for d in build/var_*; do GACT_LIB_PATH=$d/libgact.so python tools/qtime.py --dtypes bf16; done
