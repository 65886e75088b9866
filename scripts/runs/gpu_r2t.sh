timeout 600 python -m pytest tests/test_gpu_mma.py -x -q -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_pytest.log
