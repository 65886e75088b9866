bash scripts/quick2.sh 2>&1 | tail -4
B="python bench.py --config 2 --steps 1 --warmup 1 --n-iter 20 --no-e2e --no-cpu --no-dhr"
$B > gpurun_out/plain6.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist" -s 1 -c 1 -o gpurun_out/prof_persist_c2 $B > gpurun_out/ncu6.log 2>&1
tail -1 gpurun_out/ncu6.log
