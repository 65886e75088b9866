timeout 900 python -m pytest tests -q -m gpu 2>&1 | grep -E "passed|failed|Error|assert" | head -8
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b2.log 2>&1; tail -1 gpurun_out/b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', '%.4g'%d['value'], 'fbp_s', d['stages']['fbp_s'], 'dhr', d['gpu_dhr'])"
timeout 300 python bench.py --config 4 --steps 1 --warmup 1 --n-iter 2 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', 'fbp_s', d['stages']['fbp_s'], 'dhr', d['gpu_dhr'])"
B="python bench.py --steps 1 --warmup 1 --n-iter 2 --no-e2e --no-cpu"
$B > gpurun_out/plain_d.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dhr2.csv $B > gpurun_out/ncu_d.log 2>&1
echo rc=$?
