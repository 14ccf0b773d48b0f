"""A/B of the fused RMSNorm kernels of two builds of the library at the 0.5B
shape (M=16384, d=896; RMS_M / RMS_D override): python scripts/rms_ab.py A.so B.so.  20 launches per
CUDA graph, 5 interleaved rounds, median per launch; outputs compared bitwise."""
import ctypes as C
import sys

import torch

import os
M, d = int(os.environ.get("RMS_M", 16384)), int(os.environ.get("RMS_D", 896))  # 7B: RMS_M=8192 RMS_D=4096
libs = [C.CDLL(p) for p in sys.argv[1:]]
bf = lambda *s: (torch.randn(*s, device="cuda") * 0.5).to(torch.bfloat16)
nr, dy, ex, gam, res, x = bf(M, d), bf(M, d), bf(M, d), bf(d) + 1, bf(M, d), bf(M, d)
slot = torch.zeros(4, dtype=torch.int32, device="cuda")
V = lambda t: C.c_void_p(t.data_ptr())
outs, cases = [], []


class Eager:  # RMS_EAGER=1: 20 stream launches instead of a graph replay
    def __init__(self, fn):
        self.fn = fn

    def replay(self):
        for _ in range(20):
            self.fn(torch.cuda.current_stream().cuda_stream)


def graph(fn):
    if os.environ.get("RMS_EAGER"):
        fn(torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        return Eager(fn)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            fn(torch.cuda.current_stream().cuda_stream)
    return g


for i, L in enumerate(libs):
    L.qtk_rmsnorm_bwd_partials.restype = C.c_int
    part = torch.empty((L.qtk_rmsnorm_bwd_partials(C.c_int64(M), C.c_int(d)), d), device="cuda")
    din = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    dg = torch.empty(d, device="cuda")
    nro, nd = torch.empty(M, d, device="cuda", dtype=torch.bfloat16), torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    inv = torch.empty(M, device="cuda")
    bw = lambda s, L=L, part=part, din=din, dg=dg: L.qtk_rmsnorm_bwd(
        V(nr), V(gam), C.c_int64(M), C.c_int(d), C.c_float(1e-6), V(dy), V(ex), V(din), V(part), V(dg), V(slot),
        C.c_void_p(s))
    fw = lambda s, L=L, nro=nro, nd=nd, inv=inv: L.qtk_rmsnorm_fwd(
        V(x), V(res), V(gam), C.c_int64(M), C.c_int(d), C.c_float(1e-6), V(nro), V(nd), V(inv), V(slot), C.c_void_p(s))
    cases.append((i, "bwd", graph(bw)))
    cases.append((i, "fwd", graph(fw)))
    outs.append((din, dg, nd))
times = {(i, n): [] for i, n, _ in cases}
for _ in range(5):
    for i, n, g in cases:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        times[(i, n)].append(e0.elapsed_time(e1) / 20 * 1e3)
for i, n, _ in cases:
    print(f"{sys.argv[1 + i]:40s} rms_{n}: {sorted(times[(i, n)])[2]:7.1f} us")
for k in range(1, len(outs)):
    print("bitwise equal (d_in, dgamma, normed):", [torch.equal(a, b) for a, b in zip(outs[0], outs[k])])
