timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf or fhr" 2>&1 | tail -2
bash scripts/ab.sh default libhsnct_head.so
