# session 4: P1 address fold + full-mask sigma_V shuffles -- parity and C5/C3 A/B vs the previous build
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_mma.py tests/test_gpu_counts.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s4/micro_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/micro_pytest.log
tail -3 gpurun_out/s4/micro_pytest.log
P=$PWD/paper_2410_22500_b200/build/libhsnct_prev.so
for rep in 1 2 3; do
  echo "== new"; timeout 600 python scripts/tc_perf.py 5 40 mma 2>&1 | grep -v "^plans"
  echo "== prev"; HSNCT_LIB=$P timeout 600 python scripts/tc_perf.py 5 40 mma 2>&1 | grep -v "^plans"
done > gpurun_out/s4/ab_micro.txt 2>&1
cat gpurun_out/s4/ab_micro.txt
