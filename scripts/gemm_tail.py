"""Tail-split GEMM check at the 0.5B bench shapes: the auto path (split_k=0: head of whole
M panels + split-K tail when the last round is at most half full) against the single
launch (split_k=1) — ulp distance of the outputs and device time of each."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_15306_b200 import ops

torch.manual_seed(0)
T, d, F = 16384, 896, 9728
u8 = lambda r, c: torch.randint(0, 120, (r, c), dtype=torch.uint8, device="cuda")
sa = torch.tensor([3.0], device="cuda")
sb = torch.tensor([5.0], device="cuda")
res = (torch.randn(T, d, device="cuda") * 4).to(torch.bfloat16)
acc0 = (torch.randn(F, d, device="cuda") * 1e-2).to(torch.bfloat16)
cases = [
    ("gate_up wgrad (MN,MN)", dict(a=u8(T, F), b=u8(T, d), M=F, N=d, K=T, a_mn=True, b_mn=True, a_fmt=1)),
    ("gate_up wgrad SR-acc", dict(a=u8(T, F), b=u8(T, d), M=F, N=d, K=T, a_mn=True, b_mn=True, a_fmt=1,
                                  epi=ops.EPI_BF16_ACC, sr=(7, 11, 123456))),
    ("down fwd +res (K,K)", dict(a=u8(T, F // 2), b=u8(d, F // 2), M=T, N=d, K=F // 2, epi=ops.EPI_BF16_RES, res=res)),
    ("gate_up dgrad (K,MN)", dict(a=u8(T, F), b=u8(F, d), M=T, N=d, K=F, b_mn=True, a_fmt=1)),
]


def ulp(x, y):
    xi = x.view(torch.int16).cpu().numpy().astype(np.int32)
    yi = y.view(torch.int16).cpu().numpy().astype(np.int32)
    return np.abs(xi - yi)


for name, kw in cases:
    outs, times = [], []
    for sk in (1, 0):
        def f():
            o = acc0.clone() if kw.get("epi") == ops.EPI_BF16_ACC else None
            return ops.gemm(a_scale=sa, b_scale=sb, split_k=sk, out=o, **kw)
        out = f()
        torch.cuda.synchronize()
        outs.append(out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        o = acc0.clone() if kw.get("epi") == ops.EPI_BF16_ACC else torch.empty_like(out)
        g = lambda: ops.gemm(a_scale=sa, b_scale=sb, split_k=sk, out=o, **kw)
        g()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            g()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 20 * 1e3)
    du = ulp(outs[0], outs[1])
    plan = ops.gemm_plan(a_scale=sa, b_scale=sb, split_k=0, **{k: v for k, v in kw.items()})
    print(f"{name:24s} single {times[0]:7.1f} us  tail-split {times[1]:7.1f} us  exact {np.mean(du == 0):.5f} "
          f"max ulp {du.max()} le1 {np.mean(du <= 1):.6f} plan {plan}", flush=True)
