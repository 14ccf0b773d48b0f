"""Wgrad GEMM (D[out][in] = sum_m A[m][out] B[m][in], K = tokens) at the Llama-7B and
0.5B shapes: operand majorness (MN-major as stored by the forward, or K-major =
transposed copies) x epilogue (SR accumulate vs plain bf16)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops
for tag, (m_out, n_in, K) in (("7b gate_up", (22016, 4096, 8192)), ("7b down", (4096, 11008, 8192)),
                             ("7b qkv", (12288, 4096, 8192)), ("0.5b gate_up", (9728, 896, 16384))):
    for amn in (1, 0):
        for bmn in (1, 0):
            mk = lambda r, c: torch.randint(0, 120, (r, c), dtype=torch.uint8, device="cuda")
            a = mk(K, m_out) if amn else mk(m_out, K)
            b = mk(K, n_in) if bmn else mk(n_in, K)
            out = torch.zeros(m_out, n_in, dtype=torch.bfloat16, device="cuda")
            for epi in (3, 0):
                kw = dict(M=m_out, N=n_in, K=K, a_mn=bool(amn), b_mn=bool(bmn), a_fmt=1, epi=epi, out=out,
                          sr=(1, 2, 3), split_k=1)
                try:
                    plan = ops.gemm_plan(a, b, **kw)
                    f = lambda: ops.gemm(a, b, **kw)
                    f(); torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(5): f()
                    e1.record(); torch.cuda.synchronize()
                    us = e0.elapsed_time(e1) / 5 * 1e3
                    print(f"{tag:12s} a_mn={amn} b_mn={bmn} epi={'acc' if epi == 3 else 'bf16'} cg={plan['cg']} "
                          f"bn={plan['bn']} {us:8.1f} us {2.0 * m_out * n_in * K / us / 1e6:7.1f} TF/s", flush=True)
                except Exception as e:  # noqa: BLE001
                    print(f"{tag:12s} a_mn={amn} b_mn={bmn} epi={epi}: {str(e)[:100]}", flush=True)
            del a, b, out
