timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "nmf_parity or fallback" > gpurun_out/pytest_k12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k12.log
