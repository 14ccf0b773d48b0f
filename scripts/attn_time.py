"""Device time of the attention forward and backward at the bench shapes (CUDA events,
20 launches after warm-up); FA-convention causal FLOPs (fwd 4*B*H*T^2/2*hd, bwd 2.5x)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops

for name, (B, T, H, Hkv, hd) in (("0.5b", (16, 1024, 14, 2, 64)), ("7b", (8, 1024, 32, 32, 128))):
    d = H * hd
    qkv = torch.randn(B * T, d + 2 * Hkv * hd, device="cuda").to(torch.bfloat16)
    dout = (torch.randn(B * T, d, device="cuda") * 0.1).to(torch.bfloat16)
    out, out32, lse, _ = ops.attn_fwd(qkv, B, T, H, Hkv, hd)

    def t(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    fl = 4.0 * B * H * T * T / 2 * hd
    tf = t(lambda: ops.attn_fwd(qkv, B, T, H, Hkv, hd))
    tb = t(lambda: ops.attn_bwd(qkv, out32, dout, lse, B, T, H, Hkv, hd))
    print(f"{name}: fwd {tf * 1e3:.1f} us {fl / tf / 1e9:.0f} TF/s | bwd {tb * 1e3:.1f} us {2.5 * fl / tb / 1e9:.0f} TF/s",
          flush=True)
