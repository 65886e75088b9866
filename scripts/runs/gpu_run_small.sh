timeout 300 python scripts/trace_nmf.py --config 1 2>&1 | tail -25
timeout 300 python scripts/trace_nmf.py --config 2 2>&1 | tail -25
