timeout 900 python -m pytest tests/test_gpu_counts.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "stream or counts" > gpurun_out/r2s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_pytest.log
timeout 1200 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo "bench rc=$?" >> gpurun_out/r2s_bench.err
