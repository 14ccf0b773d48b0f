"""One attention forward + backward at a bench shape (for ncu --set full captures):
python scripts/attn_prof.py [0.5b|7b]."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import ops

shape = {"0.5b": (16, 1024, 14, 2, 64), "7b": (8, 1024, 32, 32, 128)}[sys.argv[1] if len(sys.argv) > 1 else "0.5b"]
B, T, H, Hkv, hd = shape
d = H * hd
qkv = torch.randn(B * T, d + 2 * Hkv * hd, device="cuda").to(torch.bfloat16)
dout = (torch.randn(B * T, d, device="cuda") * 0.1).to(torch.bfloat16)
for _ in range(2):
    out, out32, lse, _ = ops.attn_fwd(qkv, B, T, H, Hkv, hd)
    ops.attn_bwd(qkv, out32, dout, lse, B, T, H, Hkv, hd)
torch.cuda.synchronize()
print("ok")
