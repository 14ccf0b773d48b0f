"""Tiny on-device check used by __graft_entry__.smoke()."""
from __future__ import annotations

import numpy as np
import torch


def run() -> None:
    from . import ops
    assert torch.cuda.is_available(), "smoke needs cuda:0"
    torch.cuda.set_device(0)
    g = np.random.default_rng(0)
    x = g.uniform(-2, 2, (256, 512)).astype(np.float32)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    slot = ops.absmax(xt)
    codes, scale = ops.quantize(xt, ops.E4M3, slot)
    out = ops.gemm(codes, codes, M=256, N=256, K=512, a_scale=scale, b_scale=scale)
    torch.cuda.synchronize()
    xb = xt.float()
    ref = xb @ xb.T
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    assert rel < 5e-2, rel
    print(f"smoke ok: fp8 gemm rel err vs fp32 {rel:.3e}")
