timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf or fhr" 2>&1 | tail -2
B4="python bench.py --config 4 --steps 1 --warmup 1 --n-iter 3 --no-e2e --no-cpu --no-dhr"
$B4 > gpurun_out/plain_c4b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist" -s 1 -c 1 -o gpurun_out/prof_c4_v1 $B4 > gpurun_out/ncu_c4b.log 2>&1
echo "c4 rc=$?"
B2="python bench.py --config 2 --steps 1 --warmup 1 --n-iter 20 --no-e2e --no-cpu --no-dhr"
$B2 > gpurun_out/plain_c2c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist" -s 1 -c 1 -o gpurun_out/prof_c2_v1 $B2 > gpurun_out/ncu_c2c.log 2>&1
echo "c2 rc=$?"
