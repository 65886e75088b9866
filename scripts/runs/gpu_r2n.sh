timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2n_pytest.log
timeout 900 python bench.py > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; echo "bench rc=$?" >> gpurun_out/r2n_bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r2n_ref.json 2> gpurun_out/r2n_ref.err; echo "ref rc=$?" >> gpurun_out/r2n_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2n_smoke.log
