# FBP kernels at C4: plain run, then one ncu --set full capture of k_ramp and k_backproject
B4="python bench.py --config 4 --steps 1 --warmup 1 --n-iter 2 --no-e2e --no-cpu --no-dhr --no-fmd"
$B4 > gpurun_out/plain_fbp4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_ramp|k_backproject" -s 2 -c 2 -o gpurun_out/prof_fbp4b $B4 > gpurun_out/ncu_fbp4.log 2>&1
echo "fbp rc=$?"
tail -2 gpurun_out/plain_fbp4.log | cut -c1-400
