#!/bin/bash
# One GPU round trip: parity tests, smoke, a short bench and an ncu launch list.
# Usage (from this container):  gpurun --timeout 1500 -- bash tools/gpu_check.sh [quick]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
[ -f paper_2206_11357_b200/libgact.so ] || make -j8 lib
make oracle > /dev/null
echo "== pytest -m gpu" 
timeout 1200 python -m pytest tests -m gpu -q --maxfail=25 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
echo "== smoke"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke.log
if [ "$1" != "quick" ]; then
  echo "== bench"
  timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 $OUT/bench.log
  echo "== ncu launch list"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"quantize|dequantize" -c 40 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1; echo "ncu rc=$?"
fi
