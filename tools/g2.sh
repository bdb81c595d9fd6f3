mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streamthr.py -m gpu -x -q > gpurun_out/t_st.log 2>&1; echo rc=$? >> gpurun_out/t_st.log
timeout 300 python tools/quick_time.py C2 C1 > gpurun_out/q_st.log 2>&1
ATKG_ST_SLOT=16384 ATKG_ST_NS=4 timeout 300 python tools/quick_time.py C2 >> gpurun_out/q_st.log 2>&1
ATKG_ST_CTAS=1 ATKG_ST_NS=4 timeout 300 python tools/quick_time.py C2 >> gpurun_out/q_st.log 2>&1
