"""Tile-shape sweep for the short-K / narrow-N FP8 GEMMs of the 0.5B step (bn 128 vs 256, CTA pair or not)."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops
M = 16384
SH = [("fwd_qkv", M, 1152, 896, 0, 0), ("fwd_o", M, 896, 896, 0, 0), ("dgrad_o", M, 896, 896, 0, 1),
      ("dgrad_qkv", M, 896, 1152, 0, 1), ("fwd_down", M, 896, 4864, 0, 0), ("dgrad_gu", M, 896, 9728, 0, 1)]
one = torch.ones(1, device="cuda")
for name, m, n, k, amn, bmn in SH:
    u8 = lambda r, c: torch.randint(0, 120, (r, c), dtype=torch.uint8, device="cuda")
    a = u8(k, m) if amn else u8(m, k)
    b = u8(k, n) if bmn else u8(n, k)
    out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    res = []
    for bn in (0, 128, 256):
        f = lambda: ops.gemm(a, b, M=m, N=n, K=k, a_mn=bool(amn), b_mn=bool(bmn), out=out, a_scale=one, b_scale=one, bn=bn)
        try:
            f(); torch.cuda.synchronize()
        except Exception as e:
            res.append(f"bn{bn}:err"); continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res.append(f"bn{bn or 'auto'} {ms*1e3:6.1f}us {2*m*n*k/ms/1e9:7.0f}TF")
    print(f"{os.environ.get('QTB_GEMM_CG','cg-auto')} {name:10s} " + " | ".join(res), flush=True)
