set -x
nvidia-smi --query-gpu=name,memory.used,memory.total --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?" >> gpurun_out/bench_c5.err
