#!/bin/bash
cd "$(dirname "$0")/.."
make oracle > /dev/null
python tools/dbg_generic.py 96; python tools/dbg_generic.py 1056
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py -m gpu -q -p no:cacheprovider -k "generic or padding or tiny" > gpurun_out/pytest_m.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_m.log | tail -1; grep "^FAILED" gpurun_out/pytest_m.log | head
