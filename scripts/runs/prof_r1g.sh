# final-kernel ncu --set full captures at C4 (NMF 3 iterations, ramp, backprojection, synthesis)
B4="python bench.py --config 4 --steps 1 --warmup 1 --n-iter 3 --no-e2e --no-cpu --no-dhr --no-fmd"
$B4 > gpurun_out/plain_c4h.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist" -c 1 -o gpurun_out/prof_c4_r1final_c $B4 > gpurun_out/ncu_c4h.log 2>&1
echo "c4 rc=$?"
