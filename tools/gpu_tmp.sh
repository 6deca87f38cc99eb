cd /root/repo
GACT_LIB_PATH=build/var_fb2/libgact.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
bash tools/gpu_variants_q.sh
bash tools/gpu_variants_bench.sh
