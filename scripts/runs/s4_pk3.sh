# session 4: the same C6r full-iteration parity on the build before the packed block (drift comparison), FFMA plan too
mkdir -p gpurun_out/s4
HSNCT_LIB=$PWD/paper_2410_22500_b200/build/libhsnct_prev.so timeout 1500 python -m pytest tests/test_gpu_fulliter.py -m gpu -x -q -s -p no:cacheprovider -k "C6r" > gpurun_out/s4/fulliter_c6r_prev.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/fulliter_c6r_prev.log
tail -5 gpurun_out/s4/fulliter_c6r_prev.log
