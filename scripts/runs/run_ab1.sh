timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf or fhr" 2>&1 | tail -2
bash scripts/ab.sh libhsnct_base.so libhsnct_hoist.so default
HSNCT_ROTATE=1 bash scripts/ab.sh default
