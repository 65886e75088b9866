for c in 1 2 3 4 5; do
  n=20; [ $c -le 2 ] && n=200
  timeout 300 python scripts/tc_perf.py $c $n mma,ffma >> gpurun_out/mma4_perf.txt 2>&1
done
