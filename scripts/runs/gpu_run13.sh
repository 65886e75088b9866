timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q -p no:cacheprovider > gpurun_out/pytest_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sharded.log
