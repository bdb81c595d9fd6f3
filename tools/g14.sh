mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C2 C5 > gpurun_out/q_v.log 2>&1
ATKG_LIB=build/libatkg_v3.so timeout 300 python tools/quick_time.py C2 C5 >> gpurun_out/q_v.log 2>&1
ATKG_LIB=build/libatkg_v4.so timeout 300 python tools/quick_time.py C2 C5 >> gpurun_out/q_v.log 2>&1
ATKG_LIB=build/libatkg_v3.so ATKG_ST_STEP=16384 timeout 300 python tools/quick_time.py C2 >> gpurun_out/q_v.log 2>&1
