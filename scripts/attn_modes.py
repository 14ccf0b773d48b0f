"""Attention precision-mode experiment: parity vs reference + speed per mode."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from oracle import ref
from paper_2512_15306_b200 import ops, _lib
from tests.helpers import rng_floats
def ulp(a, b):
    ai = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64) >> 16
    bi = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64) >> 16
    return np.abs(ai - bi)
def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)
B, T, H, Hkv, hd = 1, 256, 4, 2, 64
d = H * hd; q = d + 2 * Hkv * hd
qkv = rng_floats(7, B * T * q, -1.5, 1.5).reshape(B * T, q)
go = rng_floats(8, B * T * d, -1, 1).reshape(B * T, d)
rows = qkv
q3 = rows[:, :d].reshape(T, H, hd).transpose(1, 0, 2); k3 = rows[:, d:d+Hkv*hd].reshape(T, Hkv, hd).transpose(1, 0, 2)
v3 = rows[:, d+Hkv*hd:].reshape(T, Hkv, hd).transpose(1, 0, 2)
o_ref = ref.sdpa(q3, k3, v3).transpose(1, 0, 2).reshape(T, d)
dq, dk, dv = ref.sdpa_backward(q3, k3, v3, go.reshape(T, H, hd).transpose(1, 0, 2))
qt = torch.from_numpy(qkv).cuda().bfloat16(); gt = torch.from_numpy(go).cuda().bfloat16()
# big timing problem: 0.5B attention shape per layer
Bb, Tb, Hb, Hkvb = 16, 1024, 14, 2
qkv_big = torch.randn(Bb * Tb, Hb * 64 + 2 * Hkvb * 64, device="cuda").bfloat16()
go_big = torch.randn(Bb * Tb, Hb * 64, device="cuda").bfloat16()
for fast in (0, 1):
    for split in (1, 0):
        _lib.lib().qtk_attn_set_mode(fast, split)
        out, out32, lse, _ = ops.attn_fwd(qt, B, T, H, Hkv, hd)
        o = out.float().cpu().numpy()
        g = ops.attn_bwd(qt, out32, gt, lse, B, T, H, Hkv, hd).float().cpu().numpy()
        gq = g[:, :d].reshape(T, H, hd).transpose(1, 0, 2)
        gk = g[:, d:d+Hkv*hd].reshape(T, Hkv, hd).transpose(1, 0, 2)
        gv = g[:, d+Hkv*hd:].reshape(T, Hkv, hd).transpose(1, 0, 2)
        res = [f"fast={fast} split={split}: fwd exact {(ulp(o, o_ref)==0).mean():.5f}"]
        for nm, x, y in (("dq", gq, dq), ("dk", gk, dk), ("dv", gv, dv)):
            res.append(f"{nm} rel {rel(x, y):.2e} exact {(ulp(x, y)==0).mean():.4f} <=1ulp {(ulp(x, y)<=1).mean():.4f}")
        ob, o32b, lseb, _ = ops.attn_fwd(qkv_big, Bb, Tb, Hb, Hkvb, 64)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(5): ops.attn_fwd(qkv_big, Bb, Tb, Hb, Hkvb, 64)
        e[1].record()
        for _ in range(5): ops.attn_bwd(qkv_big, o32b, go_big, lseb, Bb, Tb, Hb, Hkvb, 64)
        e[2].record(); torch.cuda.synchronize()
        res.append(f"fwd {e[0].elapsed_time(e[1])/5:.3f} ms bwd {e[1].elapsed_time(e[2])/5:.3f} ms")
        print(" | ".join(res))
