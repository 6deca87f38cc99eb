#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/gpu_check.sh r01e
bash tools/gpu_bench_all.sh r01e
