mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C3 C3r99 > gpurun_out/q_ilp.log 2>&1
echo "== ILP2" >> gpurun_out/q_ilp.log
ATKG_LIB=build/libatkg_ilp2.so timeout 300 python tools/quick_time.py C3 C3r99 >> gpurun_out/q_ilp.log 2>&1
echo "== R2" >> gpurun_out/q_ilp.log
ATKG_ROWRES_R=2 timeout 300 python tools/quick_time.py C3 >> gpurun_out/q_ilp.log 2>&1
