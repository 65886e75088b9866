for rep in 1 2; do for lib in default libhsnct_head.so; do
  if [ "$lib" = default ]; then unset HSNCT_LIB; else export HSNCT_LIB=$PWD/paper_2410_22500_b200/$lib; fi
  for c in 2 3; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --n-iter 1 --no-e2e --no-cpu --no-dhr --no-fmd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C$c', 'nmf(1 it incl yplus) us %.1f'%d['stages']['nmf_per_iter_us'])"
  done
done; done
unset HSNCT_LIB
