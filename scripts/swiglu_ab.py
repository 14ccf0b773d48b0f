"""A/B of the SwiGLU kernels of two builds of the library at the 0.5B shape
(M=16384, F=9728): python scripts/swiglu_ab.py A.so B.so.  Each case is 20
launches in a CUDA graph, 5 interleaved rounds, median per launch; the outputs
of the two builds are compared bitwise."""
import ctypes as C
import sys

import torch

M, F = 16384, 9728
libs = [C.CDLL(p) for p in sys.argv[1:]]
for L in libs:
    for f in ("qtk_swiglu_fwd", "qtk_swiglu_bwd"):
        getattr(L, f).restype = C.c_int
gu = (torch.randn(M, F, device="cuda") * 2).to(torch.bfloat16)
dh = torch.randn(M, F // 2, device="cuda").to(torch.bfloat16)
slot = torch.zeros(4, dtype=torch.int32, device="cuda")
outs = []


def graph(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            fn(torch.cuda.current_stream().cuda_stream)
    return g


cases = []
for i, L in enumerate(libs):
    h = torch.empty(M, F // 2, device="cuda", dtype=torch.bfloat16)
    dgu = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    fw = lambda s, L=L, h=h: L.qtk_swiglu_fwd(C.c_void_p(gu.data_ptr()), C.c_int64(M), C.c_int(F // 2),
                                              C.c_void_p(h.data_ptr()), C.c_void_p(slot.data_ptr()), C.c_void_p(s))
    bw = lambda s, L=L, d=dgu: L.qtk_swiglu_bwd(C.c_void_p(gu.data_ptr()), C.c_void_p(dh.data_ptr()), C.c_int64(M),
                                                C.c_int(F // 2), C.c_void_p(d.data_ptr()),
                                                C.c_void_p(slot.data_ptr()), C.c_void_p(s))
    cases.append((i, "fwd", graph(fw), 3 * M * F))
    cases.append((i, "bwd", graph(bw), 5 * M * F))
    outs.append((h, dgu))
times = {(i, n): [] for i, n, _, _ in cases}
for _ in range(5):
    for i, n, g, _ in cases:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        times[(i, n)].append(e0.elapsed_time(e1) / 20 * 1e3)
for i, n, _, nb in cases:
    t = sorted(times[(i, n)])[2]
    print(f"{sys.argv[1 + i]:40s} swiglu_{n}: {t:7.1f} us  {nb / t / 1e3:6.0f} GB/s")
for k in range(1, len(outs)):
    print("fwd bitwise equal:", torch.equal(outs[0][0], outs[k][0]), " bwd bitwise equal:", torch.equal(outs[0][1], outs[k][1]))
