set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
B="python bench.py --steps 1 --warmup 3 --n-iter 10 --no-e2e --no-cpu --no-dhr"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 200 --csv --log-file gpurun_out/launches_v1.csv $B > gpurun_out/ncu.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_vstep|k_bpart|k_dupdate" -s 12 -c 3 -o gpurun_out/prof_v1 $B > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
