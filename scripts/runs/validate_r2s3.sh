# round-2 session-3 validation: full GPU suite, smoke, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/v3_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/v3_pytest.txt 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/v3_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err; echo "bench rc=$?"
cat gpurun_out/v3_bench.json
