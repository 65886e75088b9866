# round 1 final-kernel evidence: launch list of the default bench command, full ncu captures
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-dhr"
$B > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv $B > gpurun_out/ncu_l.log 2>&1
echo "launches rc=$?"
B2="python bench.py --config 2 --steps 1 --warmup 1 --n-iter 20 --no-e2e --no-cpu --no-dhr"
$B2 > gpurun_out/plain_c2f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist|k_yplus|k_synth|k_ramp|k_backproject" -s 5 -c 5 -o gpurun_out/prof_c2_final $B2 > gpurun_out/ncu_c2f.log 2>&1
echo "c2 rc=$?"
B4="python bench.py --config 4 --steps 1 --warmup 1 --n-iter 3 --no-e2e --no-cpu --no-dhr"
$B4 > gpurun_out/plain_c4f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist|k_ramp|k_backproject|k_synth" -s 4 -c 4 -o gpurun_out/prof_c4_final $B4 > gpurun_out/ncu_c4f.log 2>&1
echo "c4 rc=$?"
