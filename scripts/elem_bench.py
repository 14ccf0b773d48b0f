"""Microbenchmark of the memory-bound kernels at the 0.5B step shapes (M=16384, d=896, F=9728).
Each case is captured 20x into a CUDA graph (no host overhead) with preallocated buffers."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import _lib

L = _lib.lib()
M, d, F = 16384, 896, 9728
bf = lambda *s: (torch.randn(*s, device="cuda") * 0.5).to(torch.bfloat16)
res, x, dy, ex, gam, out, out2 = bf(M, d), bf(M, d), bf(M, d), bf(M, d), bf(d), bf(M, d), bf(M, d)
gu, dh, h, dgu = bf(M, F), bf(M, F // 2), bf(M, F // 2), bf(M, F)
inv = torch.empty(M, device="cuda")
slot = torch.zeros(4, dtype=torch.int32, device="cuda")
part = torch.empty((L.qtk_rmsnorm_bwd_partials(M, d), d), device="cuda")
dg = torch.empty(d, device="cuda")
codes = torch.empty(M * F, dtype=torch.uint8, device="cuda")
sc = torch.empty(4, device="cuda")
big = bf(M, F)
P = lambda t: t.data_ptr() if t is not None else None


def t(name, f, nbytes, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f(s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            f(s.cuda_stream)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{name:28s} {us:8.1f} us  {nbytes / us / 1e3:7.0f} GB/s", flush=True)


t("rmsnorm_fwd (pass-through)", lambda s: L.qtk_rmsnorm_fwd(None, P(res), P(gam), M, d, 1e-6, None, P(out), P(inv), P(slot), s), 4 * M * d)
t("rmsnorm_fwd (x + res)", lambda s: L.qtk_rmsnorm_fwd(P(x), P(res), P(gam), M, d, 1e-6, P(out2), P(out), P(inv), P(slot), s), 8 * M * d)
t("rmsnorm_bwd", lambda s: L.qtk_rmsnorm_bwd(P(res), P(gam), M, d, 1e-6, P(dy), None, P(out), P(part), P(dg), P(slot), s), 6 * M * d)
t("rmsnorm_bwd (+extra)", lambda s: L.qtk_rmsnorm_bwd(P(res), P(gam), M, d, 1e-6, P(dy), P(ex), P(out), P(part), P(dg), P(slot), s), 8 * M * d)
t("swiglu_fwd", lambda s: L.qtk_swiglu_fwd(P(gu), M, F // 2, P(h), P(slot), s), 3 * M * F)
t("swiglu_bwd", lambda s: L.qtk_swiglu_bwd(P(gu), P(dh), M, F // 2, P(dgu), P(slot), s), 5 * M * F)
slot[1] = 0x40000000
amx = slot[1:2]
for n in (M * d, M * F):
    t(f"quantize n={n}", lambda s: L.qtk_quantize_bf16(P(big), n, 0, P(amx), P(codes), P(sc), s), 3 * n)
