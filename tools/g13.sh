mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:st_finish -s 2 -c 1 -o gpurun_out/prof_fin -f python tools/quick_time.py C2 > gpurun_out/ncu_fin.log 2>&1
