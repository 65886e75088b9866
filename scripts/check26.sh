for rot in 1 0 1 0; do
 export HSNCT_ROTATE=$rot
 for c in 4 3; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --n-iter 20 --no-e2e --no-cpu --no-dhr --no-fmd > gpurun_out/b$c.log 2>&1; tail -1 gpurun_out/b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rot $rot C$c', '%.4g'%d['value'], 'nmf/iter us %.2f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/b$c.log
 done
done
