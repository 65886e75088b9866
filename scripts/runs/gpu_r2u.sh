timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2u_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2u_smoke.log
timeout 600 python bench.py --config 6 --steps 1 --warmup 1 --no-e2e --no-cpu --no-fmd --no-mbir --no-counts > gpurun_out/r2u_c6.json 2> gpurun_out/r2u_c6.err; echo "c6 rc=$?" >> gpurun_out/r2u_c6.err
