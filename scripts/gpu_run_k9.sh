timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf" 2>&1 | tail -3
timeout 600 python scripts/tc_perf.py 6 5 ffma,twopass 2>&1 | tail -6
