timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fulliter.py -x -q 2>&1 | tail -2
timeout 600 python scripts/tc_perf.py 6 30 ffma 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_nmf_persist -c 1 -o gpurun_out/persist_c6 python scripts/tc_perf.py 6 3 ffma > gpurun_out/ncu_c6.log 2>&1; tail -2 gpurun_out/ncu_c6.log
