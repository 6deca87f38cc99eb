#!/bin/bash
# GPU tests + compute-sanitizer (memcheck / racecheck / initcheck / synccheck) over the parity
# subset that reaches every kernel family, the 2-rank gloo bench path and the reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
TAG=${1:-r01}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
     -k "c1_config or tiny_and_ragged or edge_values or batch_equals_single or group_stats_matches or threshold_ties or concurrent" > gpurun_out/sanitizer_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_${tool}_$TAG.log | tail -2
done
echo "== torchrun 2 ranks (gloo) on one GPU"
GACT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --workload bert_layer \
  --no-e2e > gpurun_out/bench_2rank_gloo_$TAG.log 2>&1; echo "rc=$?"; tail -c 400 gpurun_out/bench_2rank_gloo_$TAG.log
echo "== reference arm"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_$TAG.log 2>&1; echo "rc=$?"; tail -c 400 gpurun_out/bench_reference_$TAG.log
