mkdir -p gpurun_out
timeout 1200 python scripts/nblk_sweep.py 1,2 200 > gpurun_out/nblk_sweep.txt 2>&1; echo "rc=$?"
cat gpurun_out/nblk_sweep.txt
