timeout 300 python scripts/trace_nmf.py --config 2 --n-iter 20 2>&1 | tail -15
timeout 300 python scripts/trace_nmf.py --config 4 --n-iter 6 2>&1 | tail -15
