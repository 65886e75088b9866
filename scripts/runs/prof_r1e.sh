# launch list of the default bench command (ncu gpu__time_duration, cold-cache, serialised)
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-dhr --no-fmd"
$B > gpurun_out/plain_l2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final3.csv $B > gpurun_out/ncu_l2.log 2>&1
echo "launches rc=$?"
