HSNCT_TRACE=1 timeout 300 python scripts/trace_nmf.py --config 1 --n-iter 40 > gpurun_out/r2m_trace_c1.txt 2>&1
HSNCT_TRACE=1 timeout 300 python scripts/trace_nmf.py --config 2 --n-iter 40 > gpurun_out/r2m_trace_c2.txt 2>&1
