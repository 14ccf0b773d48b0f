"""GEMM layout experiment at the Llama-7B gate_up shapes (M=8192 tokens, F=22016, d=4096):
fwd (K,K), dgrad (K,MN), wgrad (MN,MN) with the accumulate epilogue and with a plain bf16 store."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops

T, F, d = 8192, 22016, 4096
u8 = lambda r, c: torch.randint(0, 120, (r, c), dtype=torch.uint8, device="cuda")
one = torch.ones(1, device="cuda")
cases = [
    ("fwd  (K,K)  bf16", dict(a=u8(T, d), b=u8(F, d), M=T, N=F, K=d)),
    ("dgrad(K,MN) bf16", dict(a=u8(T, F), b=u8(F, d), M=T, N=d, K=F, b_mn=True)),
    ("wgrad(MN,MN) acc", dict(a=u8(T, F), b=u8(T, d), M=F, N=d, K=T, a_mn=True, b_mn=True, epi=ops.EPI_BF16_ACC,
                              out=torch.zeros(F, d, dtype=torch.bfloat16, device="cuda"), sr=(1, 2, 3))),
    ("wgrad(MN,MN) bf16", dict(a=u8(T, F), b=u8(T, d), M=F, N=d, K=T, a_mn=True, b_mn=True)),
    ("wgrad(K,K) via copies bf16", dict(a=u8(F, T), b=u8(d, T), M=F, N=d, K=T)),
]
for name, kw in cases:
    f = lambda: ops.gemm(a_scale=one, b_scale=one, **kw)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:28s} {ms:7.3f} ms {2*T*F*d/ms/1e9:8.1f} TFLOP/s", flush=True)
