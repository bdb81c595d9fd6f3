mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C3 C3k8 C2 C5 > gpurun_out/q_default.log 2>&1
ATKG_ROWTHR=1 timeout 300 python tools/quick_time.py C3 C3k2 C3r99 > gpurun_out/q_thr.log 2>&1
ATKG_ROWTHR=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_threshold -s 3 -c 1 -o gpurun_out/prof_thr4 -f python tools/quick_time.py C3 > gpurun_out/ncu_thr.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_resident -s 3 -c 1 -o gpurun_out/prof_row4 -f python tools/quick_time.py C3 > gpurun_out/ncu_row.log 2>&1
