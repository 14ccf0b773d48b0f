"""Attention operand precision A/B (bf16 hi+lo vs bf16 P / dS): parity against the
reference sdpa / sdpa_backward (src/tensorops.cpp:191-303) and device time at the
0.5B (GQA 14/2, hd 64) and Llama-7B (MHA 32/32, hd 128) bench shapes."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from oracle import ref
from paper_2512_15306_b200 import ops, _lib
from tests.helpers import bf16_grid_round


def ulp(a, b):
    ai = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64) >> 16
    bi = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64) >> 16
    return np.abs(ai - bi)


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def parity(B, T, H, Hkv, hd, seed=1):
    d = H * hd; q = d + 2 * Hkv * hd
    g = np.random.default_rng(seed)
    qkv = bf16_grid_round((g.random(B * T * q, dtype=np.float32) * 3 - 1.5).reshape(B * T, q))
    go = bf16_grid_round((g.random(B * T * d, dtype=np.float32) * 2 - 1).reshape(B * T, d))
    qt = torch.from_numpy(qkv).cuda().to(torch.bfloat16)
    out, out32, lse, _ = ops.attn_fwd(qt, B, T, H, Hkv, hd)
    dq_ = ops.attn_bwd(qt, out32, torch.from_numpy(go).cuda().to(torch.bfloat16), lse, B, T, H, Hkv, hd)
    o = out.float().cpu().numpy()[:T, :d].reshape(T, H, hd).transpose(1, 0, 2)
    gq = dq_.float().cpu().numpy()[:T]
    grp = H // Hkv
    kv = 0
    hs = slice(0, grp)
    q3 = qkv[:T, :d].reshape(T, H, hd).transpose(1, 0, 2)[hs]
    k3 = qkv[:T, d:d + Hkv * hd].reshape(T, Hkv, hd).transpose(1, 0, 2)[kv:kv + 1]
    v3 = qkv[:T, d + Hkv * hd:].reshape(T, Hkv, hd).transpose(1, 0, 2)[kv:kv + 1]
    want = ref.sdpa(q3, k3, v3)
    u = ulp(o[hs], want)
    dq, dk, dv = ref.sdpa_backward(q3, k3, v3, go[:T].reshape(T, H, hd).transpose(1, 0, 2)[hs])
    gdq = gq[:, :d].reshape(T, H, hd).transpose(1, 0, 2)[hs]
    gdk = gq[:, d:d + Hkv * hd].reshape(T, Hkv, hd).transpose(1, 0, 2)[kv:kv + 1]
    gdv = gq[:, d + Hkv * hd:].reshape(T, Hkv, hd).transpose(1, 0, 2)[kv:kv + 1]
    res = f"o exact {(u == 0).mean():.4f} <=1 {(u <= 1).mean():.5f} max {u.max()}"
    for nm, x, y in (("dq", gdq, dq), ("dk", gdk, dk), ("dv", gdv, dv)):
        uu = ulp(x, y)
        res += f" | {nm} rel {rel(x, y):.2e} exact {(uu == 0).mean():.4f} <=1 {(uu <= 1).mean():.5f}"
    return res


def timing(B, T, H, Hkv, hd):
    d = H * hd; q = d + 2 * Hkv * hd
    qkv = torch.randn(B * T, q, device="cuda").bfloat16()
    go = torch.randn(B * T, d, device="cuda").bfloat16()
    o, o32, lse, _ = ops.attn_fwd(qkv, B, T, H, Hkv, hd)
    for _ in range(3):
        ops.attn_fwd(qkv, B, T, H, Hkv, hd); ops.attn_bwd(qkv, o32, go, lse, B, T, H, Hkv, hd)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(10): ops.attn_fwd(qkv, B, T, H, Hkv, hd)
    e[1].record()
    for _ in range(10): ops.attn_bwd(qkv, o32, go, lse, B, T, H, Hkv, hd)
    e[2].record(); torch.cuda.synchronize()
    fl = 4.0 * B * H * T * T / 2 * hd
    tf, tb = e[0].elapsed_time(e[1]) / 10, e[1].elapsed_time(e[2]) / 10
    return f"fwd {tf:.3f} ms ({fl / tf / 1e9:.0f} TF/s)  bwd {tb:.3f} ms ({2.5 * fl / tb / 1e9:.0f} TF/s)"


for plo in (1, 0):
    _lib.lib().qtk_attn_set_plo(plo)
    print(f"plo={plo} 0.5B  T=1024:", parity(1, 1024, 14, 2, 64), flush=True)
    print(f"plo={plo} 7B    T=1024:", parity(1, 1024, 32, 32, 128), flush=True)
    print(f"plo={plo} 0.5B timing (B16):", timing(16, 1024, 14, 2, 64), flush=True)
    print(f"plo={plo} 7B   timing (B8):", timing(8, 1024, 32, 32, 128), flush=True)
