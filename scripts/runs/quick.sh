timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['value'], d['stages'], d['roofline']['frac'])"
timeout 300 python bench.py --config 4 --steps 2 --warmup 3 --n-iter 20 --no-e2e --no-cpu --no-dhr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4(20it)', d['value'], d['stages'], d['roofline']['frac'])"
