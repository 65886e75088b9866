# session 4: phase-2 V operand split once per tile (vfrag_s) -- parity and A/B vs the previous build (HSNCT_LIB)
mkdir -p gpurun_out/s4
timeout 1500 python -m pytest tests/test_gpu_mma.py tests/test_gpu_parity.py tests/test_gpu_counts.py tests/test_gpu_fulliter.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s4/split_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/split_pytest.log
tail -3 gpurun_out/s4/split_pytest.log
P=$PWD/paper_2410_22500_b200/build/libhsnct_prev.so
for rep in 1 2; do
  echo "== new"; timeout 600 python scripts/tc_perf.py 6 30 mma,mma8 2>&1 | grep -v "^plans"
  echo "== prev"; HSNCT_LIB=$P timeout 600 python scripts/tc_perf.py 6 30 mma,mma8 2>&1 | grep -v "^plans"
  echo "== new"; timeout 600 python scripts/tc_perf.py 5 40 mma 2>&1 | grep -v "^plans"
  echo "== prev"; HSNCT_LIB=$P timeout 600 python scripts/tc_perf.py 5 40 mma 2>&1 | grep -v "^plans"
done > gpurun_out/s4/ab_split.txt 2>&1
cat gpurun_out/s4/ab_split.txt
