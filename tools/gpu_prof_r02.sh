#!/bin/bash
# Round-2 profiles: wave-count variants, ncu launch list of the bench step, ncu --set full of
# the bf16 quantize kernel (bench class launch and a single 2^28 tensor), summarised on the box
# (the .ncu-rep files stay there: gpurun copies back <= 64 MiB).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/ncu
OUT=gpurun_out; TAG=${1:-r02a}
for v in default w4 w16; do
  lib=paper_2206_11357_b200/libgact.so; [ $v != default ] && lib=build/var_$v/libgact.so
  [ -f $lib ] || continue
  GACT_LIB_PATH=$lib python tools/qtime.py --dtypes bf16
  GACT_LIB_PATH=$lib python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v resnet50', d['value'], d['phases']['quantize_frac'], d['phases']['dequantize_frac'])"
done
[ "$2" = "noncu" ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"quantize|dequantize" --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/ncu_bench_$TAG.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quantize_big" -s 4 -c 1 \
    -o /tmp/ncu/bench_q_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu q rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quantize_big" -s 1 -c 1 \
   -o /tmp/ncu/prof_q_$TAG -f python tools/prof_kernels.py --bits 4 --reps 2 > /dev/null 2>&1; echo "ncu q1 rc=$?"
for r in bench_q prof_q; do
  python tools/ncu_summary.py /tmp/ncu/${r}_$TAG.ncu-rep > $OUT/${r}_${TAG}_summary.txt 2>&1
  python tools/ncu_opcodes.py /tmp/ncu/${r}_$TAG.ncu-rep 30 > $OUT/${r}_${TAG}_opcodes.txt 2>&1
  ncu -i /tmp/ncu/${r}_$TAG.ncu-rep --page details --csv > $OUT/${r}_${TAG}_details.csv 2>&1
done
ls -la $OUT
