timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
HSNCT_NO_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -k "nmf or fhr" -x -q 2>&1 | tail -2
for c in 2 4; do
 n=""; [ $c = 4 ] && n="--n-iter 20"
 timeout 300 python bench.py --config $c --steps 3 --warmup 3 $n --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c', '%.3g'%d['value'], 'nmf/iter us %.1f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], 'launches', d['gpu_launches'])"
 HSNCT_NO_PERSIST=1 timeout 300 python bench.py --config $c --steps 3 --warmup 3 $n --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c nopersist', '%.3g'%d['value'], 'nmf/iter us %.1f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'])"
done
