# session 4: the final library at the paper shape: C6r full-iteration parity and the C6 bench
mkdir -p gpurun_out/s4
timeout 1500 python -m pytest tests/test_gpu_fulliter.py -m gpu -x -q -s -p no:cacheprovider -k "C6r" > gpurun_out/s4/fulliter_c6r_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/fulliter_c6r_final.log
tail -6 gpurun_out/s4/fulliter_c6r_final.log
timeout 900 python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu --no-fmd --no-counts --mbir-iters 20 > gpurun_out/s4/bench_c6_final.json 2> gpurun_out/s4/bench_c6_final.err; echo "c6 rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/s4/bench_c6_final.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'], d['stages']['nmf_per_iter_us'], d['clocks'])
print(json.dumps(d.get('mbir',{}).get('table2')))
PY
