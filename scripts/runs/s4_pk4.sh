# session 4: packed single column block for K <= 4 -- parity and C1/C2 A/B (mma plan) vs the previous build and vs FFMA
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_mma.py tests/test_gpu_parity.py tests/test_gpu_counts.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s4/pk4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/pk4_pytest.log
tail -8 gpurun_out/s4/pk4_pytest.log
P=$PWD/paper_2410_22500_b200/build/libhsnct_prev.so
for rep in 1 2; do
  for c in 2 1; do
  echo "== new C$c"; timeout 600 python scripts/tc_perf.py $c 200 mma,ffma 2>&1 | grep -v "^plans"
  echo "== prev C$c"; HSNCT_LIB=$P timeout 600 python scripts/tc_perf.py $c 200 mma 2>&1 | grep -v "^plans"
  done
done > gpurun_out/s4/ab_pk4.txt 2>&1
cat gpurun_out/s4/ab_pk4.txt
