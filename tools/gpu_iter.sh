#!/bin/bash
# One tuning iteration on the GPU: the parity files (single, batched, staged, fuzz) against the
# oracle, then tools/gpu_ab.sh (variants vs the in-tree library). Extra group sizes for the
# single-tensor timings in GS (e.g. GS="512 1024 2048").
# Usage: tools/gpu_iter.sh TAG "variants" [bench workloads...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=$1; VARS=$2; shift 2
make oracle > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider > gpurun_out/parity_$TAG.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/parity_$TAG.log; grep FAILED gpurun_out/parity_$TAG.log | head -5
for g in $GS; do for v in default $VARS; do
  L=""; [ $v != default ] && L=build/var_$v/libgact.so
  GACT_LIB_PATH=$L timeout 300 python tools/qtime.py --G $g --tag $v
done; done
tools/gpu_ab.sh $TAG "$VARS" "$@"
