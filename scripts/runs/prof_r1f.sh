# final-kernel ncu --set full captures (C2: every hot-path kernel; NMF with 20 iterations)
B2="python bench.py --config 2 --steps 1 --warmup 1 --n-iter 20 --no-e2e --no-cpu --no-dhr --no-fmd"
$B2 > gpurun_out/plain_c2h.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist|k_yplus|k_synth|k_ramp|k_backproject" -s 5 -c 5 -o gpurun_out/prof_c2_r1final $B2 > gpurun_out/ncu_c2h.log 2>&1
echo "c2 rc=$?"
