timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "synth or fhr or linearity" 2>&1 | tail -2
for lib in default libhsnct_head.so default libhsnct_head.so; do
 for c in 2 4; do
  if [ "$lib" = default ]; then unset HSNCT_LIB; else export HSNCT_LIB=$PWD/paper_2410_22500_b200/$lib; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --n-iter 2 --no-e2e --no-cpu --no-fmd --no-dhr 2>&1 | tail -1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages']; print('$lib C$c', 'synth ms %.3f frac %.3f'%(1e3*s['synth_s'], s['synth_roofline']['frac']))"
 done
done
unset HSNCT_LIB
