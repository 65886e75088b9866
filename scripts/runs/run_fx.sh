timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf or fhr" 2>&1 | tail -4
python scripts/trace_nmf.py --config 2 --n-iter 30 2>&1 | grep -E "pass_mean|dupd |bar1|bar2_restage|iter_wall"
bash scripts/ab.sh libhsnct_head.so default
