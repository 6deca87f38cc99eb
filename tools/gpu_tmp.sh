#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/gpu_check.sh r01d
bash tools/gpu_bench_all.sh r01d
