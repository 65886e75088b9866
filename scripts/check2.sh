set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "nmf or fhr" 2>&1 | tail -5
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', '%.4g'%d['value'], 'nmf/iter us %.2f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], d['clocks'])"
timeout 300 python bench.py --config 4 --steps 2 --warmup 3 --n-iter 20 --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4(20it)', '%.4g'%d['value'], 'nmf/iter us %.1f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], d['clocks'])"
timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --n-iter 20 --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3(20it)', '%.4g'%d['value'], 'nmf/iter us %.1f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], d['clocks'])"
