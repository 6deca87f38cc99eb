cd /root/repo
for d in build/var_*; do echo "== $d"; for dt in bf16; do for b in 4 1; do GACT_LIB_PATH=$d/libgact.so python tools/prof_kernels.py --bits $b --dtype $dt --reps 1 2>&1 | tail -1; done; done; done
