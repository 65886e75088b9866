# session 4: full-iteration parity at the reduced paper shape (K = 9, 300 iterations) and the C6 bench with the packed block
mkdir -p gpurun_out/s4
timeout 1500 python -m pytest tests/test_gpu_fulliter.py -m gpu -x -q -s -p no:cacheprovider -k "C6r" > gpurun_out/s4/fulliter_c6r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/fulliter_c6r.log
tail -8 gpurun_out/s4/fulliter_c6r.log
timeout 900 python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu --no-fmd --no-counts --mbir-iters 20 > gpurun_out/s4/bench_c6_pk.json 2> gpurun_out/s4/bench_c6_pk.err; echo "c6 rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/s4/bench_c6_pk.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['stages']['nmf_per_iter_us'], d['clocks'])
print(json.dumps(d.get('mbir',{}).get('table2')))
PY
