#!/bin/bash
# ncu --set full of one kernel regex on the single-tensor driver: tools/gpu_prof1.sh TAG REGEX BITS DTYPE [LIB]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
[ -n "$5" ] && export GACT_LIB_PATH=$5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 1 -c 1 \
   -o gpurun_out/prof_$1 -f python tools/prof_kernels.py --bits ${3:-4} --dtype ${4:-bf16} --reps 2 > gpurun_out/prof_$1.log 2>&1
echo "ncu rc=$?"
