mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:st_finish -s 2 -c 1 -o gpurun_out/prof_fin5 -f python tools/quick_time.py C5 > gpurun_out/ncu_fin5.log 2>&1
