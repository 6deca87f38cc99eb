#!/bin/bash
cd "$(dirname "$0")/.."
make oracle >/dev/null
timeout 900 python -m pytest tests/test_gpu_bench.py -q -p no:cacheprovider 2>&1 | tail -15
