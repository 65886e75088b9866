# Round-end style measurement: the default bench line (C5), the reference arm, the launch list of
# a short bench run and one full ncu capture of the dominant kernel.
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_c5.json 2> gpurun_out/bench_ref_c5.err; echo "rc=$?" >> gpurun_out/bench_ref_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-fmd > gpurun_out/ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_nmf_persist -c 1 -f -o gpurun_out/ncu_persist_c5 python scripts/tc_perf.py 5 2 ffma > gpurun_out/ncu_persist.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_persist.log
