mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_limits.py tests/test_abi.py -q > gpurun_out/limits_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/limits_pytest.txt
