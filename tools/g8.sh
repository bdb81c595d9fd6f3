mkdir -p gpurun_out
ATKG_LIB=build/libatkg_dbg.so timeout 300 python - > gpurun_out/dbg.log 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import torch, paper_2506_04165_b200 as atk
for shape, B, kp, k in [((1, 1<<30), 256, 8, 1024), ((256, 262144), 128, 2, 64)]:
    x = torch.randn(*shape, device='cuda')
    p = atk.AlgoParams(shape[1], B, kp, k)
    v, i = atk.approx_top_k_device(x, p)
    torch.cuda.synchronize()
    print("done", shape)
PY
timeout 900 python -m pytest tests/test_gpu_streamthr.py -m gpu -x -q > gpurun_out/t_st.log 2>&1; echo rc=$? >> gpurun_out/t_st.log
timeout 300 python tools/quick_time.py C2 C5 > gpurun_out/q_st.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:st_ --csv python tools/quick_time.py C2 C5 > gpurun_out/st_launch.csv 2>&1
