mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C3 C3k8 > gpurun_out/q_rk.log 2>&1
echo "== rank emit at 512" >> gpurun_out/q_rk.log
ATKG_LIB=build/libatkg_rk256.so timeout 300 python tools/quick_time.py C3 C3k8 >> gpurun_out/q_rk.log 2>&1
