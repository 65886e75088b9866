timeout 1500 python -m pytest tests/test_gpu_fullsize.py -v -x 2>&1 | grep -E "PASS|FAIL|Error|assert|SKIP|passed|failed|rel" | head -20
