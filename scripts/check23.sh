timeout 600 python scripts/sanitize.py > gpurun_out/san_plain.log 2>&1 && timeout 1200 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python scripts/sanitize.py > gpurun_out/memcheck.log 2>&1
echo rc=$?
tail -5 gpurun_out/memcheck.log
