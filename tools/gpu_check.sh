#!/bin/bash
# One GPU round trip: parity tests (incl. full-size), smoke, the bench, an ncu launch list
# of the bench command and ncu --set full captures of the two hot kernels.
# Usage (from this container):  gpurun --timeout 2400 -- bash tools/gpu_check.sh [tag]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
TAG=${1:-r01}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
[ -f paper_2206_11357_b200/libgact.so ] || make -j8 lib
make oracle > /dev/null
echo "== pytest -m gpu"
timeout 1800 python -m pytest tests -m gpu -q --maxfail=25 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
echo "== smoke"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
echo "== bench"
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -c 2500 $OUT/bench_$TAG.log
echo "== ncu launch list"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"quantize|dequantize" --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_bench_$TAG.log 2>&1; echo "ncu rc=$?"
echo "== ncu --set full (first quantize / dequantize launch of a bench step)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quantize_big" -s 4 -c 1 \
    -o $OUT/bench_q_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu q rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dequantize" -s 4 -c 1 \
    -o $OUT/bench_d_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu d rc=$?"
