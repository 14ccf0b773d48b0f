"""bf16 GEMM rate: the product's tcgen05 kind::f16 GEMM vs cuBLAS (torch.matmul) at 8192^3 and at
the LM-head shapes of the 0.5B step (M=16384 tokens, d=896, V=151936), CUDA events, best of 5x10."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps / 1e3)
    return best


for name, M, N, K, a_mn, b_mn, epi in (("8192^3 KK", 8192, 8192, 8192, False, False, 0),
                                        ("8192^3 K,MN", 8192, 8192, 8192, False, True, 0),
                                        ("lm fwd logits", 16384, 151936, 896, False, False, 1),
                                        ("lm dgrad", 16384, 896, 151936, False, True, 1),
                                        ("lm wgrad", 151936, 896, 16384, True, True, 1)):
    a = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(device="cuda", dtype=torch.bfloat16)
    b = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
    kw = dict(M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out, split_k=0)
    plan = ops.gemm_plan(a, b, **kw)
    ours = t(lambda: ops.gemm(a, b, **kw))
    A = a.t() if a_mn else a
    B = b if b_mn else b.t()
    cub = t(lambda: torch.matmul(A, B))
    fl = 2.0 * M * N * K
    print(f"{name:14s} ours {fl / ours / 1e12:7.1f} TF/s ({ours * 1e3:.2f} ms, {plan})  cuBLAS {fl / cub / 1e12:7.1f} TF/s",
          flush=True)
