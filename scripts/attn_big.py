"""0.5B-shape attention fwd+bwd once (for ncu)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops
B, T, H, Hkv, hd = 16, 1024, 14, 2, 64
qkv = torch.randn(B * T, H * hd + 2 * Hkv * hd, device="cuda").bfloat16()
go = torch.randn(B * T, H * hd, device="cuda").bfloat16()
for _ in range(2):
    o, o32, lse, _ = ops.attn_fwd(qkv, B, T, H, Hkv, hd)
    ops.attn_bwd(qkv, o32, go, lse, B, T, H, Hkv, hd)
torch.cuda.synchronize()
