#!/bin/bash
# Bench lines for every BASELINE.json config (C2 sweep, C3, C4, C5) on one GPU.
# Usage: gpurun --timeout 1800 -- bash tools/gpu_bench_all.sh [tag]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r01}
make oracle > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
OUT=gpurun_out/bench_all_$TAG.jsonl; : > $OUT
timeout 900 python bench.py --steps 10 --warmup 3 2>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT
for w in buf256 bert_layer bert24 gcn_swin; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --cpu-seconds 3 2>>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT
done
for b in 1 2 4 8; do
  timeout 600 python bench.py --workload buf256 --avg-bits $b --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT
done
timeout 600 python bench.py --dtype f32 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT
