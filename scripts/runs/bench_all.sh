# round-1 bench lines for every BASELINE config at its full iteration count (C1 is the small
# oracle-sized case); one JSON line each into gpurun_out/bench_C*.json
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_C$c.json 2> gpurun_out/bench_C$c.err
  echo "C$c rc=$?"; tail -1 gpurun_out/bench_C$c.json | cut -c1-200
done
