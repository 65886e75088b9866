timeout 300 python scripts/tc_perf.py 2 400 mma,ffma > gpurun_out/r2r_c2.txt 2>&1
timeout 300 python scripts/tc_perf.py 1 400 mma,ffma > gpurun_out/r2r_c1.txt 2>&1
timeout 300 python scripts/tc_perf.py 3 40 mma,ffma > gpurun_out/r2r_c3.txt 2>&1
