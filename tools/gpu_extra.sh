#!/bin/bash
# Extra GPU evidence: the N > 1 bench path (2 ranks on one GPU over gloo), compute-sanitizer
# on the kernels, and the bench on every BASELINE.json workload. Results -> gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
TAG=${1:-r01}
echo "== torchrun 2 ranks (gloo) on one GPU"
GACT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --workload bert_layer \
  --no-e2e > gpurun_out/bench_2rank_gloo_$TAG.log 2>&1; echo "rc=$?"; tail -c 600 gpurun_out/bench_2rank_gloo_$TAG.log
echo "== reference arm"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_$TAG.log 2>&1; echo "rc=$?"; tail -c 400 gpurun_out/bench_reference_$TAG.log
echo "== workloads"
for w in buf256 bert_layer gcn_swin; do
  timeout 900 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu-baseline > gpurun_out/bench_${w}_$TAG.log 2>&1
  echo "$w rc=$?"; tail -c 300 gpurun_out/bench_${w}_$TAG.log; echo
done
timeout 900 python bench.py --steps 10 --warmup 3 --workload resnet50 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/bench_resnet50_f32_$TAG.log 2>&1
echo "resnet50 f32 rc=$?"
echo "== compute-sanitizer"
for tool in memcheck racecheck initcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
     -k "c1_config or tiny_and_ragged or edge_values or batch_equals_single or group_stats_matches" > gpurun_out/sanitizer_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_${tool}_$TAG.log | tail -2
done
