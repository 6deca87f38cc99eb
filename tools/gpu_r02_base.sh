#!/bin/bash
# Round-2 baseline: GPU tests, the bench line, per-kernel single-tensor rates.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err; echo "bench rc=$?"
cat gpurun_out/bench_base.json | head -c 1500; echo
for dt in bf16 f16 f32; do for b in 1 2 4 8; do
  python tools/prof_kernels.py --bits $b --dtype $dt --reps 1 2>&1 | tail -1
done; done
