# A/B of library builds on C2 and C4 (20 iterations): bash scripts/ab.sh lib1.so lib2.so ...
# (HSNCT_LIB selects the library; the first argument "default" means the in-tree libhsnct.so)
for rep in 1 2; do
 for lib in "$@"; do
  for c in 2 4; do
   n=""; [ $c = 4 ] && n="--n-iter 20"
   [ $c = 3 ] && n="--n-iter 20"
   if [ "$lib" = default ]; then unset HSNCT_LIB; else export HSNCT_LIB=$PWD/paper_2410_22500_b200/$lib; fi
   timeout 300 python bench.py --config $c --steps 3 --warmup 3 $n --no-e2e --no-cpu --no-dhr --no-fmd 2>&1 | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C$c', '%.4g'%d['value'], 'nmf/iter us %.1f'%d['stages']['nmf_per_iter_us'], 'hbm %.3f'%d['roofline']['frac'], 'sm', d['clocks']['sm_mhz'])"
  done
 done
done
unset HSNCT_LIB
