#!/bin/bash
# Round-2 evidence refresh after the third session's kernel changes: full GPU suite, smoke,
# the default bench line, clocked bench lines of every config, ncu launch list + full capture
# of the b = 1 and b = 4 quantize launches and the b = 4 dequantize launch of the bench step. Usage: tools/gpu_r02c.sh TAG
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02c}
mkdir -p $OUT /tmp/ncu
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi_$TAG.txt 2>&1
make oracle > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" $OUT/pytest_gpu_$TAG.log | tail -1; grep -E "^FAILED" $OUT/pytest_gpu_$TAG.log | head
cp $OUT/everygroup_counts.json $OUT/everygroup_counts_$TAG.json 2>/dev/null; cp $OUT/dequant_counts.json $OUT/dequant_counts_$TAG.json 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; head -c 600 $OUT/bench_$TAG.json; echo
A=$OUT/bench_all_$TAG.jsonl; : > $A
for w in bert_layer bert24 gcn_swin; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --cpu-seconds 3 2>>$OUT/bench_err_$TAG.log | tail -1 >> $A
done
for b in 1 2 4 8; do
  timeout 600 python bench.py --workload buf256 --avg-bits $b --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>$OUT/bench_err_$TAG.log | tail -1 >> $A
done
for dt in f32 f16; do
  timeout 600 python bench.py --dtype $dt --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>>$OUT/bench_err_$TAG.log | tail -1 >> $A
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_$TAG.log 2>&1; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"quantize|dequantize" --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/ncu_bench_$TAG.log 2>&1; echo "ncu list rc=$?"
# launch order per step: b = 4, 8, 1, 2 quantize classes, then dequantize; -s skips the warm-up
for spec in "q4:quantize_big:12" "q1:quantize_big:14" "dq4:dequantize:12"; do
  n=${spec%%:*}; r=${spec#*:}; k=${r%%:*}; s=${r#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
      -o /tmp/ncu/bench_${n}_$TAG -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $n rc=$?"
  python tools/ncu_summary.py /tmp/ncu/bench_${n}_$TAG.ncu-rep > $OUT/ncu_${n}_${TAG}_summary.txt 2>&1
  python tools/ncu_opcodes.py /tmp/ncu/bench_${n}_$TAG.ncu-rep 30 > $OUT/ncu_${n}_${TAG}_opcodes.txt 2>&1
done
# (compute-sanitizer is closed on this pool since the third session: the earlier round-2 runs,
# profiles/r02_sanitizer.md, were clean; the changed paths are covered by the parity tests.)
