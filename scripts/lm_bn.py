"""LM-head backward GEMMs (split-A, N = d = 896): BN 256 (last N tile half empty) vs 128 (no waste)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops
M, V, d = 16384, 151936, 896
bf = lambda r, c: (torch.randn(r, c, device="cuda") * 0.01).to(torch.bfloat16)
dl, dl2, W, h = bf(M, V), bf(M, V), bf(V, d), bf(M, d)
out = torch.empty(M, d, dtype=torch.bfloat16, device="cuda")
gw = torch.zeros(V, d, dtype=torch.bfloat16, device="cuda")
for name, f in [
    ("dhidden", lambda bn: ops.gemm(dl, W, M=M, N=d, K=V, b_mn=True, out=out, a2=dl2, bn=bn)),
    ("dW", lambda bn: ops.gemm(dl, h, M=V, N=d, K=M, a_mn=True, b_mn=True, epi=ops.EPI_F32_ACC, out=gw, a2=dl2, bn=bn,
                               sr=(1, 2, 0))),
]:
    for bn in (256, 128, 256, 128):
        f(bn); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): f(bn)
        e1.record(); torch.cuda.synchronize()
        print(name, bn, round(e0.elapsed_time(e1) / 3, 3), "ms", flush=True)
