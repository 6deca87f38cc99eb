#!/bin/bash
# ncu --set full captures of the quantize and dequantize kernels (one GPU).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r01}
BITS=${2:-4}
for dt in bf16 f32; do
  python tools/prof_kernels.py --bits $BITS --dtype $dt --reps 1 2>&1 | tail -1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quantize_big -s 1 -c 1 \
   -o gpurun_out/prof_q_$TAG -f python tools/prof_kernels.py --bits $BITS --reps 2 > gpurun_out/prof_q_$TAG.log 2>&1
echo "ncu q rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dequantize -s 1 -c 1 \
   -o gpurun_out/prof_d_$TAG -f python tools/prof_kernels.py --bits $BITS --reps 2 > gpurun_out/prof_d_$TAG.log 2>&1
echo "ncu d rc=$?"
