timeout 900 python -m pytest tests/test_gpu_fmd.py -v 2>&1 | grep -E "PASS|FAIL|Error|assert|passed|failed|rel" | head -20
