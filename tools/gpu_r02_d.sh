#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
timeout 1200 python -m pytest tests/test_gpu_controller.py tests/test_gpu_parity.py tests/test_gpu_bench.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_d.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_d.log
timeout 1800 python -m pytest tests/test_gpu_everygroup.py -m gpu -q -p no:cacheprovider -x -s > gpurun_out/pytest_every.log 2>&1
echo "every rc=$?"; tail -5 gpurun_out/pytest_every.log
