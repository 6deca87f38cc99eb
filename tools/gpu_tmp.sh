#!/bin/bash
# racecheck on the kernels that use shared memory (G >= 2048: per-warp stage / CTA exchange)
cd "$(dirname "$0")/.."
make oracle >/dev/null
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
   -k "(quantize_dequantize_parity and (2048 or 4096)) or (tiny_and_ragged and 2048) or group_stats_matches" > gpurun_out/sanitizer_racecheck_smem_r01c.log 2>&1
echo "racecheck rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer_racecheck_smem_r01c.log | tail -3
