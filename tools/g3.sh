mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:st_ --csv python tools/quick_time.py C2 > gpurun_out/st_launch.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:st_ -s 4 -c 2 -o gpurun_out/prof_st -f python tools/quick_time.py C2 > gpurun_out/ncu_st.log 2>&1
