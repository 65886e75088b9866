timeout 1500 python -m pytest tests/test_gpu_fullsize.py -v -x 2>&1 | grep -E "PASS|FAIL|Error|assert|SKIP|passed|failed" | head -10
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -1 gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
