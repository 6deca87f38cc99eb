cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for d in build/var_*; do echo "== $d"; for G in 2048 4096; do for dt in bf16 f16 f32; do GACT_LIB_PATH=$d/libgact.so python tools/prof_kernels.py --bits 4 --dtype $dt --G $G --reps 1 2>&1 | tail -1; done; done; done
