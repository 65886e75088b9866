# every BASELINE config (C1-C4) and the paper shape (C6) at full iteration counts, plus the reference arm at C5
mkdir -p gpurun_out/allcfg
for c in 1 2 3 4 6; do
  timeout 900 python bench.py --config $c --no-mbir --no-fmd --no-counts > gpurun_out/allcfg/bench_c$c.json 2> gpurun_out/allcfg/bench_c$c.err
  echo "c$c rc=$?"; tail -c 400 gpurun_out/allcfg/bench_c$c.json
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/allcfg/bench_ref_c5.json 2> gpurun_out/allcfg/bench_ref_c5.err; echo "ref rc=$?"
cat gpurun_out/allcfg/bench_ref_c5.json
