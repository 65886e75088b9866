timeout 900 python -m pytest tests/test_gpu_parity.py -k "nmf" -x -q 2>&1 | tail -2
timeout 300 python bench.py --config 4 --steps 2 --warmup 3 --n-iter 20 --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4(20it)', d['value'], d['stages'], d['roofline']['frac'])"
B="python bench.py --config 4 --steps 1 --warmup 1 --n-iter 4 --no-e2e --no-cpu --no-dhr"
$B > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_fused|k_dred" -s 2 -c 2 -o gpurun_out/prof_fused $B > gpurun_out/ncu3.log 2>&1
tail -2 gpurun_out/ncu3.log
