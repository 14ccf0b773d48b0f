"""fwd2q_tc_kernel (two Q tiles per CTA) vs fwd1p_tc_kernel: bitwise equality of out / out32 /
LSE / absmax on several shapes (odd tile counts, ragged T), then device time at the bench
shapes; plus the reference check of test_bench_shapes-style sampled heads."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops, _lib
L = _lib.lib()


def run(mode, qkv, B, T, H, Hkv, hd):
    L.qtk_attn_set_fwd2q(mode)
    out, out32, lse, am = ops.attn_fwd(qkv, B, T, H, Hkv, hd)
    torch.cuda.synchronize()
    return out, out32, lse, am


for (B, T, H, Hkv, hd) in ((2, 256, 4, 2, 64), (1, 384, 4, 1, 64), (2, 200, 4, 4, 128), (16, 1024, 14, 2, 64),
                           (8, 1024, 32, 32, 128), (1, 128, 2, 2, 64), (3, 640, 8, 2, 128)):
    d = H * hd
    q = d + 2 * Hkv * hd
    g = torch.Generator(device="cuda").manual_seed(T + hd)
    qkv = (torch.randn(B * T, q, device="cuda", generator=g) * 1.5).to(torch.bfloat16)
    a = run(0, qkv, B, T, H, Hkv, hd)
    b = run(1, qkv, B, T, H, Hkv, hd)
    eq = [torch.equal(x, y) for x, y in zip(a, b)]
    diff = (a[0].float() - b[0].float()).abs().max().item()
    print(f"B={B} T={T} H={H}/{Hkv} hd={hd}: equal(out, out32, lse, amax) {eq} max|dout| {diff:.3e}", flush=True)
for (B, T, H, Hkv, hd) in ((16, 1024, 14, 2, 64), (8, 1024, 32, 32, 128)):
    d = H * hd
    q = d + 2 * Hkv * hd
    qkv = torch.randn(B * T, q, device="cuda").to(torch.bfloat16)
    for mode in (0, 1):
        L.qtk_attn_set_fwd2q(mode)
        for _ in range(3):
            ops.attn_fwd(qkv, B, T, H, Hkv, hd)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            ops.attn_fwd(qkv, B, T, H, Hkv, hd)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        fl = 4.0 * B * H * T * T / 2 * hd
        print(f"mode={mode} B={B} H={H}/{Hkv} hd={hd}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.0f} TF/s", flush=True)
