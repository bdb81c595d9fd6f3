#!/bin/bash
# C4 evidence: same-run timings (plain tcgen05 GEMM, torch bf16 matmul, fused GEMM + top-k) and one
# ncu --set full capture of gemm_tc_kernel (tensor-pipe utilisation, DRAM bytes).
# usage: bash tools/prof_c4.sh <outdir>
OUT=$1; mkdir -p $OUT
python tools/c4_time.py > $OUT/c4_time.log 2>&1 || { tail -5 $OUT/c4_time.log; exit 1; }
cat $OUT/c4_time.log
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o $OUT/gemm_tc -f \
  python tools/prof_c4_target.py 5 > $OUT/ncu_c4.log 2>&1
tail -2 $OUT/ncu_c4.log
ncu -i $OUT/gemm_tc.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h,u,v=rows[0],rows[1],rows[2]
for i,n in enumerate(h):
    if any(k in n for k in ['pipe_tensor','dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','sm__throughput.avg.pct','sm__inst_executed_pipe_uniform','issue_active.avg.pct']): print(n,u[i],v[i])
" | tee $OUT/gemm_tc_metrics.txt
# tile-order A/B: panel width 1 (previous order) vs the default
python - <<PY | tee $OUT/c4_panel.log
import sys; sys.path.insert(0, ".")
import torch, paper_2506_04165_b200 as atk
from paper_2506_04165_b200 import topk as T
m, kd, n = 8192, 3584, 14336
dev = torch.device("cuda:0"); g = torch.Generator(device="cpu").manual_seed(0)
x = torch.randn((m, kd), generator=g).to(torch.bfloat16).to(dev)
w = (0.02 * torch.randn((n, kd), generator=g)).to(torch.bfloat16).to(dev)
p = atk.AlgoParams(n, 128, 4, 287); st = torch.zeros(1, dtype=torch.int32, device=dev)
out = (torch.empty((m, 287), dtype=torch.float32, device=dev), torch.empty((m, 287), dtype=torch.int32, device=dev))
def t(iters=20):
    for _ in range(3): T.fused_gemm_top_k_device(x, w, p, status=st, out=out)
    torch.cuda.synchronize(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): T.fused_gemm_top_k_device(x, w, p, status=st, out=out)
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / iters * 1e3
ref = None
for npanel in [1, 4, 8, 16, 32, None]:
    if npanel is None: atk._lib.set_option("gemm_n_panel", None)
    else: atk._lib.set_option("gemm_n_panel", npanel)
    us = t(); v = out[0].clone(); i = out[1].clone()
    same = True if ref is None else bool(torch.equal(v, ref[0]) and torch.equal(i, ref[1]))
    ref = ref or (v, i)
    print(f"n_panel={npanel}: fused gemm+top-k {us:8.1f} us, same results {same}", flush=True)
PY
