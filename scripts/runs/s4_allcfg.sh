# session 4: every BASELINE config (C1-C4) at full iteration counts on the final library
mkdir -p gpurun_out/s4/allcfg
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --no-mbir --no-fmd --no-counts > gpurun_out/s4/allcfg/bench_c$c.json 2> gpurun_out/s4/allcfg/bench_c$c.err
  echo "c$c rc=$?"
  python - <<PY
import json
d=json.load(open('gpurun_out/s4/allcfg/bench_c$c.json'))
print('C$c', '%.4g'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'nmf frac %.3f'%d['roofline']['frac'], 'nmf/iter us %.1f'%d['stages']['nmf_per_iter_us'], 'synth %.3f'%d['stages']['synth_hbm_frac'], 'dhr %.3g'%(d['gpu_dhr']['value'] if d.get('gpu_dhr') else 0), 'e2e %.3g'%(d['e2e']['value'] if d.get('e2e') else 0), 'cpu %.3g'%(d['cpu_baseline']['value'] if d.get('cpu_baseline') else 0), d['clocks']['sm_mhz'])
PY
done
