#!/bin/bash
# Round-2 evidence run: full GPU suite (incl. every-group parity at full size), smoke, the
# bench line, ncu launch list + full capture of the quantize kernel (summarised on the box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/ncu
OUT=gpurun_out; TAG=${1:-r02}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi_$TAG.txt 2>&1
make oracle > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" $OUT/pytest_gpu_$TAG.log | tail -1; grep -E "^FAILED" $OUT/pytest_gpu_$TAG.log | head
cp $OUT/everygroup_counts.json $OUT/everygroup_counts_$TAG.json 2>/dev/null; cp $OUT/dequant_counts.json $OUT/dequant_counts_$TAG.json 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; head -c 3000 $OUT/bench_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"quantize|dequantize" --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/ncu_bench_$TAG.log 2>&1; echo "ncu list rc=$?"
for k in quantize_big dequantize; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 4 -c 1 \
      -o /tmp/ncu/bench_${k}_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $k rc=$?"
  python tools/ncu_summary.py /tmp/ncu/bench_${k}_$TAG.ncu-rep > $OUT/ncu_${k}_${TAG}_summary.txt 2>&1
  python tools/ncu_opcodes.py /tmp/ncu/bench_${k}_$TAG.ncu-rep 30 > $OUT/ncu_${k}_${TAG}_opcodes.txt 2>&1
done
