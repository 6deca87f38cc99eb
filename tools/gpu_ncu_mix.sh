#!/bin/bash
# ncu --set full of the b = 4 and b = 1 quantize launches of one bench step (ResNet-50 bf16)
# and their instruction mixes. Usage: tools/gpu_ncu_mix.sh TAG
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=$1; mkdir -p $OUT /tmp/ncu
for spec in "q4:12" "q1:14"; do
  n=${spec%%:*}; s=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quantize_big -s $s -c 1 \
      -o /tmp/ncu/bench_${n}_$TAG -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $n rc=$?"
  python tools/ncu_summary.py /tmp/ncu/bench_${n}_$TAG.ncu-rep > $OUT/ncu_${n}_${TAG}_summary.txt 2>&1
  python tools/ncu_opcodes.py /tmp/ncu/bench_${n}_$TAG.ncu-rep 40 > $OUT/ncu_${n}_${TAG}_opcodes.txt 2>&1
done
