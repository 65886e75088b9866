timeout 600 python -m pytest tests/test_gpu_mma.py -x -q -p no:cacheprovider -k "timing" > gpurun_out/r2h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc=$?" >> gpurun_out/r2h_bench.err
