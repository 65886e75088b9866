# session 4: phase-2 skip-last-dummy-block experiment (libhsnct_skiplast.so, -DHSNCT_MMA_SKIPLAST) vs the product build
mkdir -p gpurun_out/s4
X=$PWD/paper_2410_22500_b200/libhsnct_skiplast.so
HSNCT_LIB=$X timeout 600 python -m pytest tests/test_gpu_mma.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2 3; do
  echo "== product C5"; timeout 600 python scripts/tc_perf.py 5 40 mma 2>&1 | grep -v "^plans"
  echo "== skiplast C5"; HSNCT_LIB=$X timeout 600 python scripts/tc_perf.py 5 40 mma 2>&1 | grep -v "^plans"
done > gpurun_out/s4/ab_skiplast.txt 2>&1
for rep in 1 2; do
  echo "== product C6"; timeout 600 python scripts/tc_perf.py 6 30 mma 2>&1 | grep -v "^plans"
  echo "== skiplast C6"; HSNCT_LIB=$X timeout 600 python scripts/tc_perf.py 6 30 mma 2>&1 | grep -v "^plans"
done >> gpurun_out/s4/ab_skiplast.txt 2>&1
cat gpurun_out/s4/ab_skiplast.txt
