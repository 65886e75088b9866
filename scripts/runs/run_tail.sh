timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf or fhr" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
python scripts/trace_nmf.py --config 4 --n-iter 6 2>&1 | grep -E "pass_mean|iter_wall"
bash scripts/ab.sh libhsnct_head.so default
