cd /root/repo
bash tools/gpu_variants_q.sh
bash tools/gpu_variants_bench.sh
