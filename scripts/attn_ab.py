"""A/B of the attention kernels of two builds of the library: python scripts/attn_ab.py A.so B.so.
Forward + backward at the 0.5B and 7B bench shapes; outputs (out, out32, lse, dqkv) compared
bitwise between the builds, device time per call (CUDA events, 20 calls, median of 5 rounds)."""
import ctypes as C
import sys

import torch

V = lambda t: C.c_void_p(t.data_ptr() if t is not None else 0)
libs = [C.CDLL(p) for p in sys.argv[1:]]
for L in libs:
    L.qtk_attn_bwd_ws_bytes.restype = C.c_size_t
for name, (B, T, H, Hkv, hd) in (("0.5b", (16, 1024, 14, 2, 64)), ("7b", (8, 1024, 32, 32, 128)),
                                 ("odd", (3, 640, 8, 2, 128)), ("gqa", (2, 384, 4, 1, 64))):
    d = H * hd
    qd = d + 2 * Hkv * hd
    g = torch.Generator(device="cuda").manual_seed(T + hd)
    qkv = (torch.randn(B * T, qd, device="cuda", generator=g)).to(torch.bfloat16)
    dout = (torch.randn(B * T, d, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    res, times = [], []
    for L in libs:
        out = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
        out32 = torch.empty(B * T, d, device="cuda")
        lse = torch.empty(B, H, T, device="cuda")
        slot = torch.zeros(1, dtype=torch.int32, device="cuda")
        Dv = torch.empty(B, H, T, device="cuda")
        dqkv = torch.zeros_like(qkv)
        ws = torch.empty(max(L.qtk_attn_bwd_ws_bytes(B, T, H, Hkv, hd) // 4, 1), device="cuda")
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        fw = lambda: L.qtk_attn_fwd(V(qkv), B, T, H, Hkv, hd, qd, V(out), C.c_int64(d), V(out32), V(lse), V(slot), s)
        bw = lambda: L.qtk_attn_bwd(V(qkv), V(out32), V(dout), C.c_int64(d), V(lse), V(Dv), B, T, H, Hkv, hd, qd,
                                    V(dqkv), V(ws), s)
        assert fw() == 0 and bw() == 0
        torch.cuda.synchronize()
        res.append([out.clone(), out32.clone(), lse.clone(), dqkv.clone()])
        tt = []
        for fn in (fw, bw):
            r = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                r.append(e0.elapsed_time(e1) / 20 * 1e3)
            tt.append(sorted(r)[2])
        times.append(tt)
    eq = [all(torch.equal(a, b) for a, b in zip(res[0], r)) for r in res[1:]]
    print(f"{name}: " + " | ".join(f"{sys.argv[1 + i].split('/')[-1]} fwd {t[0]:.1f} us bwd {t[1]:.1f} us"
                                   for i, t in enumerate(times)) + f"  bitwise equal: {eq}", flush=True)
