# session 4: K = 9..16 on 16 warps -- parity (mma / parity / counts tests) and the C6 A/B against the 8-warp form
mkdir -p gpurun_out/s4
timeout 1200 python -m pytest tests/test_gpu_mma.py tests/test_gpu_parity.py tests/test_gpu_counts.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s4/mw16_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/mw16_pytest.log
tail -3 gpurun_out/s4/mw16_pytest.log
timeout 600 python scripts/tc_perf.py 6 30 mma,mma8,mma,mma8 > gpurun_out/s4/perf_c6_mw16.txt 2>&1; echo "perf rc=$?"
cat gpurun_out/s4/perf_c6_mw16.txt
