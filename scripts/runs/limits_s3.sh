mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_limits.py tests/test_abi.py -q -x > gpurun_out/limits_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/limits_pytest.txt
timeout 900 python bench.py --config 6 --steps 2 --warmup 3 --no-fmd --no-counts --no-e2e --no-cpu --mbir-iters 20 > gpurun_out/bench_c6_t2.json 2> gpurun_out/bench_c6_t2.err; echo "c6 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c6_t2.json')); print(d['value'], d['mbir'])"
tail -3 gpurun_out/bench_c6_t2.err
