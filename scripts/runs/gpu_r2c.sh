timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
timeout 300 python scripts/tc_perf.py 5 3 mma > gpurun_out/r2c_plain.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/ncu_mma_c5 python scripts/tc_perf.py 5 3 mma > gpurun_out/ncu_mma_c5.log 2>&1
echo done
