B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dhr --no-fmd --no-mbir --no-counts"
$B > gpurun_out/r2d_plain.json 2> gpurun_out/r2d_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2d_launches_c5.csv $B > gpurun_out/r2d_ncu.log 2>&1
echo rc=$?
timeout 300 python scripts/tc_perf.py 6 5 ffma > gpurun_out/r2d_c6.txt 2>&1
cuobjdump -sass paper_2410_22500_b200/libhsnct.so > /tmp/all.sass 2>/dev/null; grep -c HMMA /tmp/all.sass > gpurun_out/r2d_sass_counts.txt
