for rep in 1 2; do
for v in default rs2 rs2_norot; do
  case $v in default) unset HSNCT_LIB; unset HSNCT_ROTATE;; rs2) export HSNCT_LIB=$PWD/paper_2410_22500_b200/libhsnct_rs2.so; unset HSNCT_ROTATE;; rs2_norot) export HSNCT_LIB=$PWD/paper_2410_22500_b200/libhsnct_rs2.so; export HSNCT_ROTATE=0;; esac
  timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-dhr --no-fmd 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'nmf/iter us %.1f'%d['stages']['nmf_per_iter_us'])"
done; done
unset HSNCT_LIB HSNCT_ROTATE
