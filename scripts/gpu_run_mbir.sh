set -x
timeout 900 python -m pytest tests/test_gpu_mbir.py -x -q -s 2>&1 | tail -30
timeout 300 python scripts/mbir_perf.py --config 5 --iters 3 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum --clock-control none --csv --log-file gpurun_out/mbir_c5_launches.csv python scripts/mbir_perf.py --config 5 --iters 2 > gpurun_out/ncu_mbir.log 2>&1
tail -3 gpurun_out/ncu_mbir.log
