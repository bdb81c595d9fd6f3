mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C2 > gpurun_out/q_ab.log 2>&1
ATKG_ST_CFAC_X=1000 timeout 300 python tools/quick_time.py C2 >> gpurun_out/q_ab.log 2>&1
ATKG_NO_PDL=1 timeout 300 python tools/quick_time.py C2 >> gpurun_out/q_ab.log 2>&1
