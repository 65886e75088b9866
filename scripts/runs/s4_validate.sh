# session-4 validation of HEAD on a fresh box: GPU tests, smoke, default bench (C5), reference arm, ncu launch list
mkdir -p gpurun_out/s4
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/s4/gpu.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=8 > gpurun_out/s4/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s4/smoke.log
( time timeout 1500 python bench.py > gpurun_out/s4/bench_c5.json 2> gpurun_out/s4/bench_c5.err ) 2> gpurun_out/s4/bench_c5.time; echo "bench rc=$?" >> gpurun_out/s4/bench_c5.err
( time timeout 900 python bench.py --impl reference > gpurun_out/s4/bench_ref.json 2> gpurun_out/s4/bench_ref.err ) 2> gpurun_out/s4/bench_ref.time; echo "ref rc=$?" >> gpurun_out/s4/bench_ref.err
tail -3 gpurun_out/s4/pytest.log; cat gpurun_out/s4/smoke.log | tail -2; cat gpurun_out/s4/bench_c5.json; cat gpurun_out/s4/bench_c5.time gpurun_out/s4/bench_ref.time
