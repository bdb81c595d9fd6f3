mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C3k1 C3k2 C3r99 C3k8 > gpurun_out/q_c3.log 2>&1
echo "== stream for short rows" >> gpurun_out/q_c3.log
ATKG_STREAMTHR_MIN_N=8192 timeout 300 python tools/quick_time.py C3k1 C3k2 C3r99 C3k8 C3 >> gpurun_out/q_c3.log 2>&1
