"""A/B of the streaming RMSNorm chain kernel's rows per CTA (QTB_CHAIN_ROWS 32 vs 16) at
the 7B (M=8192, d=4096) and 14B (M=4096, d=5120) shapes: two copies of the library, each
reading the variable at its first launch; outputs compared bitwise."""
import ctypes as C
import os
import shutil
import sys
import tempfile

import torch

src = sys.argv[1] if len(sys.argv) > 1 else "paper_2512_15306_b200/libqtrain_b200.so"
tmp = tempfile.mkdtemp()
V = lambda t: C.c_void_p(t.data_ptr())
for M, d in ((8192, 4096), (4096, 5120)):
    res = {}
    for rows in (32, 16):
        path = os.path.join(tmp, f"lib{rows}_{M}.so")
        shutil.copy(src, path)
        os.environ["QTB_CHAIN_ROWS"] = str(rows)
        L = C.CDLL(path)
        torch.manual_seed(0)
        bf = lambda *s: (torch.randn(*s, device="cuda") * 0.5).to(torch.bfloat16)
        nr, dy, ex, gam, rs, x = bf(M, d), bf(M, d), bf(M, d), bf(d) + 1, bf(M, d), bf(M, d)
        slot = torch.zeros(4, dtype=torch.int32, device="cuda")
        L.qtk_rmsnorm_bwd_partials.restype = C.c_int
        part = torch.empty((L.qtk_rmsnorm_bwd_partials(C.c_int64(M), C.c_int(d)), d), device="cuda")
        din = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
        dg = torch.empty(d, device="cuda")
        nro, nd = torch.empty_like(din), torch.empty_like(din)
        inv = torch.empty(M, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        bw = lambda: L.qtk_rmsnorm_bwd(V(nr), V(gam), C.c_int64(M), C.c_int(d), C.c_float(1e-6), V(dy), V(ex), V(din),
                                       V(part), V(dg), V(slot), C.c_void_p(s))
        fw = lambda: L.qtk_rmsnorm_fwd(V(x), V(rs), V(gam), C.c_int64(M), C.c_int(d), C.c_float(1e-6), V(nro), V(nd),
                                       V(inv), V(slot), C.c_void_p(s))
        t = {}
        for name, fn in (("bwd", bw), ("fwd", fw)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t[name] = e0.elapsed_time(e1) / 20 * 1e3
        first = (din.clone(), dg.clone(), nd.clone())
        # determinism: outputs pre-filled with garbage, recomputed, compared with the first run
        for o in (din, nd):
            o.fill_(-7.0)
        dg.fill_(float("nan"))
        part.fill_(float("nan"))
        fw()
        bw()
        torch.cuda.synchronize()
        again = [torch.equal(a_, b_) for a_, b_ in zip(first, (din, dg, nd))]
        res[rows] = (t, din.clone(), dg.clone(), nd.clone())
        print(f"M={M} d={d} rows/CTA={rows}: bwd {t['bwd']:.1f} us  fwd {t['fwd']:.1f} us  repeat-equal {again}",
              flush=True)
    a, b = res[32], res[16]
    print("  bitwise equal (d_in, dgamma, normed):", [torch.equal(x, y) for x, y in zip(a[1:], b[1:])], flush=True)
