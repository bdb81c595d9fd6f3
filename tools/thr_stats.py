"""Row-threshold path statistics (development aid; needs a library built with -DATKG_THR_STATS)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04165_b200 as atk
rows, n, B, kp, k = 8192, 14336, 128, 4, 287
x = torch.randn(rows, n, device="cuda").to(torch.bfloat16)
for r in [int(a) for a in sys.argv[1:]] or [0]:
    if r:
        os.environ["ATKG_ROWTHR_R"] = str(r)
    st = torch.zeros(8, dtype=torch.int32, device="cuda")
    atk.approx_top_k_device(x, atk.AlgoParams(n, B, kp, k), status=st)
    torch.cuda.synchronize()
    s = st.cpu().tolist()
    print(f"r={r}: slow rows {s[1]}, mean marks {s[2]/rows:.1f}, mean M {s[3]/rows:.1f}, mean large-marks {s[4]/rows:.1f}, G overflow {s[5]}")
