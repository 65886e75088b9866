timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fallback" 2>&1 | grep -E "Error|error|assert|passed|failed" | head -20
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf or fhr" 2>&1 | tail -3
for c in 2 3 4; do
 n=""; [ $c != 2 ] && n="--n-iter 20"
 timeout 300 python bench.py --config $c --steps 3 --warmup 3 $n --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c', '%.4g'%d['value'], 'nmf/iter us %.2f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], 'synth %.3f'%d['stages']['synth_hbm_frac'], d['clocks'])"
done
