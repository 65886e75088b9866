timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_project -s 1 -c 1 -o gpurun_out/proj_c5 python scripts/mbir_perf.py --config 5 --iters 2 > gpurun_out/ncu_proj.log 2>&1
tail -3 gpurun_out/ncu_proj.log
