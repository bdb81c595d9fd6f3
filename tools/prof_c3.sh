mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "rowres_ties or golden or c3" > gpurun_out/pt.log 2>&1; echo rc=$? >> gpurun_out/pt.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_resident -s 3 -c 1 -o gpurun_out/prof_C3_row4 -f python tools/quick_time.py C3 > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
