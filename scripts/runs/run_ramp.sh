for lib in default libhsnct_r3.so default libhsnct_r3.so; do
 for c in 4 3; do
  if [ "$lib" = default ]; then unset HSNCT_LIB; else export HSNCT_LIB=$PWD/paper_2410_22500_b200/$lib; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --n-iter 2 --no-e2e --no-cpu --no-fmd --no-dhr 2>&1 | tail -1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages']; print('$lib C$c', 'ramp ms %.4f frac %.3f'%(1e3*s['ramp_s'], s['ramp_roofline']['frac']))"
 done
done
