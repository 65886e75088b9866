timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "nmf or fhr" 2>&1 | grep -E "passed|failed|Error|assert" | head -3
for pf in 1 0 1 0; do
 export HSNCT_L2PF=$pf
 for c in 4 2; do
  n=""; [ $c != 2 ] && n="--n-iter 20"
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 $n --no-e2e --no-cpu --no-dhr --no-fmd > gpurun_out/b$c.log 2>&1; tail -1 gpurun_out/b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf $pf C$c', '%.4g'%d['value'], 'nmf/iter us %.2f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/b$c.log
 done
done
