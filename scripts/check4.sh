for c in 3 4; do
 timeout 300 python bench.py --config $c --steps 2 --warmup 2 --n-iter 10 --no-e2e --no-cpu --no-dhr > gpurun_out/b$c.log 2>&1; tail -4 gpurun_out/b$c.log | cut -c1-400
done
timeout 300 python scripts/trace_nmf.py --config 2 --n-iter 20 2>&1 | tail -12
timeout 300 python scripts/trace_nmf.py --config 4 --n-iter 6 2>&1 | tail -12
