for ng in 3 4; do
 export HSNCT_NGRP=$ng
 echo "== NGRP env $ng"
 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "nmf or fhr" 2>&1 | grep -E "passed|failed|Error|assert" | head -3
 timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-dhr --no-fmd > gpurun_out/b2.log 2>&1; tail -1 gpurun_out/b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', '%.4g'%d['value'], 'nmf/iter us %.2f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])"
 timeout 300 python scripts/trace_nmf.py --config 2 --n-iter 20 2>&1 | tail -9 | head -4
done
