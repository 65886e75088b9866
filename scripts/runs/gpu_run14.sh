timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_ramp_reg|k_backproject" -c 2 -f -o gpurun_out/ncu_fbp_c5 python scripts/fbp_perf.py 5 > gpurun_out/ncu_fbp.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_fbp.log
