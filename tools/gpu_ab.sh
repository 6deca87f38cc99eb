#!/bin/bash
# A/B timing of tuning variants (build/var_*/libgact.so) against the in-tree library: single
# 2^28-element tensors (tools/qtime.py) and bench lines, alternating variants, twice.
# Usage: tools/gpu_ab.sh TAG "var1 var2" [bench workloads, e.g. resnet50 bert24 buf256:1]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=$1; VARS=$2; shift 2
OUT=gpurun_out/ab_$TAG.log; : > $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader >> $OUT
lib() { if [ $1 = default ]; then echo ""; else echo build/var_$1/libgact.so; fi; }
for rep in 1 2; do
  for v in default $VARS; do
    GACT_LIB_PATH=$(lib $v) timeout 300 python tools/qtime.py --dtypes ${DTYPES:-bf16} --bits ${BITS:-1,2,4,8} --G ${G:-256} --tag $v >> $OUT 2>&1
  done
done
for rep in 1 2; do
  for w in "$@"; do
    for v in default $VARS; do
      wl=${w%%:*}; ab=""; [ "$w" != "$wl" ] && ab="--avg-bits ${w#*:}"
      GACT_LIB_PATH=$(lib $v) timeout 600 python bench.py --workload $wl $ab --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>>$OUT | tail -1 \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; c=d['clocks']; print('$w [$v]', d['value'], 'q', p['quantize_frac'], 'dq', p['dequantize_frac'], c['sm_mhz'], c['reasons'])" >> $OUT
    done
  done
done
cat $OUT
