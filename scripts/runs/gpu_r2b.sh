timeout 900 python -m pytest tests/test_gpu_mma.py tests/test_gpu_counts.py -x -q -p no:cacheprovider > gpurun_out/r2b_pytest1.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest1.log
for c in 1 2 3 5; do
  n=20; [ $c -le 2 ] && n=200
  timeout 300 python scripts/tc_perf.py $c $n mma,ffma >> gpurun_out/r2b_perf.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?" >> gpurun_out/r2b_bench.err
