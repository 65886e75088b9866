# session 4: the opt-in 16-warp form under test, C6 bench on the default (8-warp, split-once) build
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_mma.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s4/mma_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/mma_pytest.log
tail -3 gpurun_out/s4/mma_pytest.log
timeout 900 python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu --no-fmd --no-counts > gpurun_out/s4/bench_c6.json 2> gpurun_out/s4/bench_c6.err; echo "c6 rc=$?"
cat gpurun_out/s4/bench_c6.json | cut -c1-1800
