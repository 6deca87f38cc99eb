#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_l.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_l.log | tail -1; grep "^FAILED" gpurun_out/pytest_l.log | head
for G in 96 800 4064 256; do python tools/qtime.py --dtypes bf16 --G $G --bits 2,4; done
