cd /root/repo
timeout 900 python -m pytest tests/test_gpu_staged.py -x -q 2>&1 | tail -15
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1
