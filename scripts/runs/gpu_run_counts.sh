timeout 300 python scripts/counts_perf.py 3 2>&1 | tail -2
timeout 300 python scripts/counts_perf.py 5 2>&1 | tail -2
