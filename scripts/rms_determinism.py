"""Determinism of qtk_rmsnorm_fwd / _bwd: outputs of repeated launches into garbage-filled
buffers must be bitwise equal.  Shapes: RMS_SHAPES env (M:d,...)."""
import ctypes as C
import os
import sys
import pathlib
import torch
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2512_15306_b200 import _lib
L = _lib.lib()
V = lambda t: C.c_void_p(t.data_ptr())
shapes = [tuple(int(x) for x in s.split(":")) for s in os.environ.get(
    "RMS_SHAPES", "16384:896,8192:4096,4096:5120,256:5120,64:4096").split(",")]
for M, d in shapes:
    torch.manual_seed(0)
    bf = lambda *s: (torch.randn(*s, device="cuda") * 0.5).to(torch.bfloat16)
    nr, dy, ex, gam, rs, x = bf(M, d), bf(M, d), bf(M, d), bf(d) + 1, bf(M, d), bf(M, d)
    slot = torch.zeros(4, dtype=torch.int32, device="cuda")
    L.qtk_rmsnorm_bwd_partials.restype = C.c_int
    npart = L.qtk_rmsnorm_bwd_partials(C.c_int64(M), C.c_int(d))
    outs = []
    for rep in range(3):
        part = torch.full((npart, d), float("nan"), device="cuda")
        din = torch.full((M, d), -7.0, device="cuda").to(torch.bfloat16)
        dg = torch.full((d,), float("nan"), device="cuda")
        nro, nd = din.clone(), din.clone()
        inv = torch.full((M,), float("nan"), device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        rc1 = L.qtk_rmsnorm_fwd(V(x), V(rs), V(gam), C.c_int64(M), C.c_int(d), C.c_float(1e-6), V(nro), V(nd), V(inv),
                                V(slot), C.c_void_p(s))
        rc2 = L.qtk_rmsnorm_bwd(V(nr), V(gam), C.c_int64(M), C.c_int(d), C.c_float(1e-6), V(dy), V(ex), V(din),
                                V(part), V(dg), V(slot), C.c_void_p(s))
        torch.cuda.synchronize()
        outs.append((nro, nd, inv, din, dg))
    eq = [[torch.equal(a, b) for a, b in zip(outs[0], o)] for o in outs[1:]]
    nan = [bool(torch.isnan(t.float()).any()) for t in outs[0]]
    print(f"M={M} d={d} rc={rc1},{rc2} repeat-equal (nr, normed, inv, d_in, dgamma) {eq} nan {nan}", flush=True)
