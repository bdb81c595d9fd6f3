"""Counts logged vs accepted entries of the stage-1 log (debug build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2506_04165_b200 as atk
from tools.quick_time import cfgs
for name in sys.argv[1:]:
    rows, n, B, kp, k, dt = cfgs[name]
    x = torch.randn(rows, n, device="cuda")
    if dt == "bf16": x = x.to(torch.bfloat16)
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    atk.stage1_device(x, atk.AlgoParams(n, B, kp, k), status=st)
    torch.cuda.synchronize()
    s = st.cpu().tolist()
    print(f"{name}: elements={rows*n} logged={s[1]} ({s[1]/rows/n:.4f}/elem) taken={s[2]} ({s[2]/rows/n:.4f}/elem) flushes={s[3]}")
