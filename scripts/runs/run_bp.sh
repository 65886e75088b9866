timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fbp or dhr or fhr or linearity or smoke" 2>&1 | tail -2
for lib in default libhsnct_head.so; do
 for c in 2 1 3; do
  if [ "$lib" = default ]; then unset HSNCT_LIB; else export HSNCT_LIB=$PWD/paper_2410_22500_b200/$lib; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --n-iter 2 --no-e2e --no-cpu --no-fmd 2>&1 | tail -1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages']; print('$lib C$c', 'ramp ms %.4f frac %.3f'%(1e3*s['ramp_s'], s['ramp_roofline']['frac']), 'bp ms %.3f smem frac %.3f'%(1e3*s['backproject_s'], s['backproject_roofline']['frac']), 'dhr %.3g'%d['gpu_dhr']['value'])"
 done
done
unset HSNCT_LIB
