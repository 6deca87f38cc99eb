#!/bin/bash
# Clocked bench lines for every BASELINE.json config + compute-sanitizer (round 2).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r02}
make oracle > /dev/null
OUT=gpurun_out/bench_all_$TAG.jsonl; : > $OUT
timeout 900 python bench.py --steps 20 --warmup 5 2>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT | head -c 300; echo
for w in buf256 bert_layer bert24 gcn_swin; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --cpu-seconds 3 2>>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT | head -c 300; echo
done
for b in 1 2 4 8; do
  timeout 600 python bench.py --workload buf256 --avg-bits $b --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT | head -c 300; echo
done
for dt in f32 f16; do
timeout 600 python bench.py --dtype $dt --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/bench_err_$TAG.log | tail -1 | tee -a $OUT | head -c 300; echo
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_$TAG.log 2>&1; echo "reference rc=$?"
bash tools/gpu_sanitize_r02.sh $TAG
