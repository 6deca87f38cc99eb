cd /root/repo
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_staged.py -x -q -k "oracle or pageable or validation" 2>&1 | tail -5
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_staged.py -x -q -k "oracle" 2>&1 | tail -3
