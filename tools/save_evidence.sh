#!/bin/bash
# Copy one tools/gpu_r02c.sh run (gpurun_out/*_TAG*) into profiles/TAG_*: bench lines, launch list
# (and traffic.json), ncu summaries + instruction mixes, GPU suite summary. Usage: TAG "note"
cd "$(dirname "$0")/.."
TAG=$1; NOTE=$2; O=gpurun_out
python tools/make_traffic.py $O/launches_$TAG.csv resnet50 profiles/${TAG}_launches_resnet50.md > /dev/null
cp $O/bench_$TAG.json profiles/${TAG}_bench_resnet50.json
cp $O/bench_all_$TAG.jsonl profiles/${TAG}_bench_all_configs.jsonl
tail -1 $O/bench_reference_$TAG.log >> profiles/${TAG}_bench_all_configs.jsonl
{ echo "# ncu --set full summaries ($TAG; tools/gpu_r02c.sh $TAG)"; echo; echo "$NOTE"; echo
  echo '```'; cat $O/ncu_q4_${TAG}_summary.txt $O/ncu_q1_${TAG}_summary.txt $O/ncu_dq4_${TAG}_summary.txt; echo '```'; echo
  echo "Quantize instruction mix, b = 4 (7.65 M warp tiles of 256 elements in this launch):"; echo; echo '```'; cat $O/ncu_q4_${TAG}_opcodes.txt; echo '```'; echo
  echo "b = 1 (5.62 M warp tiles):"; echo; echo '```'; cat $O/ncu_q1_${TAG}_opcodes.txt; echo '```'; } > profiles/${TAG}_ncu_full.md
{ echo "# GPU suite ($TAG; tools/gpu_r02c.sh $TAG)"; echo; echo '```'; grep -E "passed|failed" $O/pytest_gpu_$TAG.log | tail -1; tail -1 $O/smoke_$TAG.log
  python3 -c "
import json; d=json.load(open('$O/everygroup_counts_$TAG.json'))
for k,v in d.items(): print('every group,', k, ':', v['elements'], 'elements,', v['code_word_mismatches'], 'code-word mismatches,', v['y_mismatches_1ulp'], 'decoded values 1 ulp from the oracle')"
  echo "dequant mismatch counts (parity tests): $(cat $O/dequant_counts_$TAG.json)"; echo '```'; } > profiles/${TAG}_gpu_suite.md
