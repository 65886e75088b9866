timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "nmf or fhr" 2>&1 | grep -E "passed|failed|Error|assert" | head -3
for c in 2 3 4; do
  n=""; [ $c != 2 ] && n="--n-iter 20"
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 $n --no-e2e --no-cpu --no-dhr --no-fmd > gpurun_out/b$c.log 2>&1; tail -1 gpurun_out/b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c', '%.4g'%d['value'], 'nmf/iter us %.2f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/b$c.log
done
timeout 300 python scripts/trace_nmf.py --config 4 --n-iter 6 2>&1 | grep -E "pass_mean|iter_wall"
timeout 300 python scripts/trace_nmf.py --config 2 --n-iter 20 2>&1 | grep -E "pass_mean|iter_wall"
