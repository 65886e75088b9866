# session 4: packed second column block (K = 9..12) -- parity and C6 A/B vs the previous build
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_mma.py tests/test_gpu_parity.py tests/test_gpu_counts.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s4/pk_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/pk_pytest.log
tail -15 gpurun_out/s4/pk_pytest.log
P=$PWD/paper_2410_22500_b200/build/libhsnct_prev.so
for rep in 1 2; do
  echo "== new"; timeout 600 python scripts/tc_perf.py 6 30 mma,mma16 2>&1 | grep -v "^plans"
  echo "== prev"; HSNCT_LIB=$P timeout 600 python scripts/tc_perf.py 6 30 mma 2>&1 | grep -v "^plans"
done > gpurun_out/s4/ab_pk.txt 2>&1
cat gpurun_out/s4/ab_pk.txt
