"""GEMM microbenchmark over the 0.5B training-step shapes (QTB_GEMM_CG env selects 1- or 2-CTA)."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops
M = 16384
SH = [  # name, kind(0 fp8/1 bf16), M, N, K, a_mn, b_mn, epi, split_a
    ("fwd_qkv", 0, M, 1152, 896, 0, 0, 0, 0), ("fwd_o", 0, M, 896, 896, 0, 0, 0, 0),
    ("fwd_gu", 0, M, 9728, 896, 0, 0, 0, 0), ("fwd_down", 0, M, 896, 4864, 0, 0, 0, 0),
    ("dgrad_down", 0, M, 4864, 896, 0, 1, 0, 0), ("dgrad_gu", 0, M, 896, 9728, 0, 1, 0, 0),
    ("dgrad_o", 0, M, 896, 896, 0, 1, 0, 0), ("dgrad_qkv", 0, M, 896, 1152, 0, 1, 0, 0),
    ("wgrad_down", 0, 896, 4864, M, 1, 1, 0, 0), ("wgrad_gu", 0, 9728, 896, M, 1, 1, 0, 0),
    ("wgrad_o", 0, 896, 896, M, 1, 1, 0, 0), ("wgrad_qkv", 0, 1152, 896, M, 1, 1, 0, 0),
    ("lm_logits", 1, M, 151936, 896, 0, 0, 1, 0), ("lm_dhidden", 1, M, 896, 151936, 0, 1, 0, 1),
    ("lm_dw", 1, 151936, 896, M, 1, 1, 1, 1),
]
cg = os.environ.get("QTB_GEMM_CG", "auto")
tot_t = 0.0
for name, kind, m, n, k, amn, bmn, epi, sa in SH:
    dt = torch.uint8 if kind == 0 else torch.bfloat16
    def mk(r, c):
        return (torch.randint(0, 120, (r, c), dtype=torch.uint8, device="cuda") if kind == 0
                else torch.randn(r, c, device="cuda").to(torch.bfloat16))
    a = mk(k, m) if amn else mk(m, k)
    b = mk(k, n) if bmn else mk(n, k)
    a2 = mk(*a.shape) if sa else None
    out = torch.empty(m, n, dtype=torch.float32 if epi == 1 else torch.bfloat16, device="cuda")
    f = lambda: ops.gemm(a, b, M=m, N=n, K=k, a_mn=bool(amn), b_mn=bool(bmn), epi=epi, out=out, a2=a2,
                         split_k=0 if (m * n) < 4e6 else 1)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3 if k * m * n > 1e12 else 10
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * m * n * k * (2 if sa else 1)
    tot_t += ms
    print(f"cg={cg} {name:12s} {ms:8.3f} ms  {fl / ms / 1e9:8.1f} TFLOP/s")
print(f"cg={cg} total {tot_t:.2f} ms")
