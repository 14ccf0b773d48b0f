"""ctypes/numpy binding of oracle/_build/liboracle.so -- the plain-C
restatement of the reference arithmetic (oracle/qtrain_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg as the checker, never on the product path.  It
travels to the GPU box (built in-tree), unlike /root/reference.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64, u64, ci, cf = C.c_int64, C.c_uint64, C.c_int, C.c_float


class _Opt:
    @classmethod
    def from_param(cls, obj):
        return None if obj is None else f32p.from_param(obj)


_SIGS = {
    "qto_f8_decode": (cf, [C.c_uint8, ci]),
    "qto_f8_encode": (C.c_uint8, [cf, ci]),
    "qto_f8_fmax": (cf, [ci]),
    "qto_absmax": (ci, [f32p, i64, C.POINTER(cf)]),
    "qto_absmax_scale": (cf, [cf, ci]),
    "qto_quantize_with_absmax": (None, [f32p, i64, ci, cf, u8p, C.POINTER(cf)]),
    "qto_transpose_quantize_with_absmax": (None, [f32p, i64, i64, ci, cf, u8p, C.POINTER(cf)]),
    "qto_fnv1a64": (u64, [C.c_char_p]),
    "qto_rng_uniform": (C.c_uint32, [u64, u64, u64]),
    "qto_rng_uniform_float": (cf, [u64, u64, u64]),
    "qto_rng_normal": (cf, [u64, u64, u64]),
    "qto_bf16_round": (cf, [cf]),
    "qto_sr_bf16": (cf, [cf, u64, u64, u64]),
    "qto_matmul_fp8": (None, [u8p, i64, i64, ci, cf, u8p, i64, ci, cf, ci, f32p]),
    "qto_matmul_f32": (None, [f32p, i64, i64, f32p, i64, ci, f32p]),
    "qto_rmsnorm_fwd": (None, [_Opt, f32p, f32p, i64, i64, cf, f32p, f32p, C.POINTER(cf)]),
    "qto_rmsnorm_bwd": (None, [f32p, f32p, i64, i64, cf, f32p, _Opt, f32p, f32p]),
    "qto_swiglu_fwd": (None, [f32p, i64, i64, f32p, C.POINTER(cf)]),
    "qto_swiglu_bwd": (None, [f32p, i64, i64, f32p, f32p]),
    "qto_sdpa_fwd": (None, [f32p, f32p, f32p, i64, i64, i64, i64, f32p]),
    "qto_sdpa_bwd": (None, [f32p, f32p, f32p, f32p, i64, i64, i64, i64, f32p, f32p, f32p]),
    "qto_embedding_backward": (ci, [i32p, i64, f32p, i64, i64, f32p]),
    "qto_cross_entropy": (ci, [f32p, i64, i64, f32p, i64, i32p, ci, C.POINTER(cf), _Opt, _Opt]),
    "qto_adamw_range": (ci, [C.c_char_p, f32p, f32p, f32p, f32p, i64, i64, i64, cf, cf, cf, cf, cf, ci, ci, u64,
                             i64, cf]),
    "qto_grad_norm_partials": (C.c_double, [f32p, i64, i64]),
    "qto_grad_accumulate": (None, [C.c_char_p, f32p, f32p, i64, ci, u64, u64]),
    "qto_init_normal": (None, [f32p, i64, cf, u64, C.c_char_p]),
    "qto_shard_layout": (None, [i64, ci, C.POINTER(i64), C.POINTER(i64)]),
}

_lib = None


def available() -> bool:
    return LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise RuntimeError(f"{LIB} not built (make -C oracle oracle)")
        l = C.CDLL(str(LIB))
        for n, (rt, at) in _SIGS.items():
            f = getattr(l, n)
            f.restype = rt
            f.argtypes = at
        _lib = l
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def f8_decode_table(kind: int) -> np.ndarray:
    return np.array([lib().qto_f8_decode(c, kind) for c in range(256)], np.float32)


def f8_encode(x, kind: int) -> np.ndarray:
    x = _f32(x).ravel()
    return np.array([lib().qto_f8_encode(float(v), kind) for v in x], np.uint8)


def absmax(x) -> float:
    x = _f32(x).ravel()
    r = cf()
    if lib().qto_absmax(x, x.size, C.byref(r)) != 0:
        raise RuntimeError("absmax: NaN element (training diverged?)")
    return r.value


def absmax_scale(a: float, kind: int) -> float:
    return lib().qto_absmax_scale(a, kind)


def quantize_with_absmax(x, kind: int, amax: float):
    x = _f32(x)
    codes = np.empty(x.size, np.uint8)
    s = cf()
    lib().qto_quantize_with_absmax(x.ravel(), x.size, kind, amax, codes, C.byref(s))
    return codes.reshape(x.shape), s.value


def transpose_quantize_with_absmax(x, kind: int, amax: float):
    x = _f32(x)
    r, c = x.shape
    codes = np.empty(r * c, np.uint8)
    s = cf()
    lib().qto_transpose_quantize_with_absmax(x, r, c, kind, amax, codes, C.byref(s))
    return codes.reshape(c, r), s.value


def rng_uniform(seed, stream, counter) -> int:
    return lib().qto_rng_uniform(seed, stream, counter)


def fnv1a64(s: str) -> int:
    return lib().qto_fnv1a64(s.encode())


def bf16_round(x: float) -> float:
    return lib().qto_bf16_round(x)


def stochastic_round_bf16(x, seed, stream, counter) -> float:
    return lib().qto_sr_bf16(x, seed, stream, counter)


def matmul_fp8(a_codes, a_kind, a_scale, b_codes, b_kind, b_scale, round_bf16=True):
    a = np.ascontiguousarray(a_codes, np.uint8)
    b = np.ascontiguousarray(b_codes, np.uint8)
    out = np.empty((a.shape[0], b.shape[0]), np.float32)
    lib().qto_matmul_fp8(a, a.shape[0], a.shape[1], a_kind, a_scale, b, b.shape[0], b_kind, b_scale, int(round_bf16),
                         out)
    return out


def matmul_f32(a, b, round_bf16=True):
    a, b = _f32(a), _f32(b)
    out = np.empty((a.shape[0], b.shape[0]), np.float32)
    lib().qto_matmul_f32(a, a.shape[0], a.shape[1], b, b.shape[0], int(round_bf16), out)
    return out


def rmsnorm_residual_fused(x, res, gamma, eps=1e-6):
    res, gamma = _f32(res), _f32(gamma)
    rows, d = res.shape
    nr, normed = np.empty_like(res), np.empty_like(res)
    am = cf()
    lib().qto_rmsnorm_fwd(None if x is None else _f32(x), res, gamma, rows, d, eps, nr, normed, C.byref(am))
    return nr, normed, am.value


def rmsnorm_residual_backward(nr, gamma, dy, d_extra=None, eps=1e-6):
    nr, gamma, dy = _f32(nr), _f32(gamma), _f32(dy)
    rows, d = nr.shape
    din, dg = np.empty_like(nr), np.empty(d, np.float32)
    lib().qto_rmsnorm_bwd(nr, gamma, rows, d, eps, dy, None if d_extra is None else _f32(d_extra), din, dg)
    return din, dg


def swiglu_fused(gu):
    gu = _f32(gu)
    h = np.empty((gu.shape[0], gu.shape[1] // 2), np.float32)
    am = cf()
    lib().qto_swiglu_fwd(gu, gu.shape[0], gu.shape[1], h, C.byref(am))
    return h, am.value


def swiglu_backward(gu, dh):
    gu, dh = _f32(gu), _f32(dh)
    out = np.empty_like(gu)
    lib().qto_swiglu_bwd(gu, gu.shape[0], gu.shape[1], dh, out)
    return out


def sdpa(q, k, v):
    q, k, v = _f32(q), _f32(k), _f32(v)
    H, T, D = q.shape
    out = np.empty_like(q)
    lib().qto_sdpa_fwd(q, k, v, H, k.shape[0], T, D, out)
    return out


def sdpa_backward(q, k, v, go):
    q, k, v, go = _f32(q), _f32(k), _f32(v), _f32(go)
    H, T, D = q.shape
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    lib().qto_sdpa_bwd(q, k, v, go, H, k.shape[0], T, D, dq, dk, dv)
    return dq, dk, dv


def embedding_backward(ids, grad_out, vocab):
    ids = np.ascontiguousarray(ids, np.int32)
    g = _f32(grad_out)
    out = np.empty((vocab, g.shape[1]), np.float32)
    if lib().qto_embedding_backward(ids, ids.size, g, g.shape[1], vocab, out) != 0:
        raise IndexError("embedding backward: token id out of range")
    return out


def cross_entropy(hidden, lm_w, targets, with_grads=True):
    h, w = _f32(hidden), _f32(lm_w)
    t = np.ascontiguousarray(targets, np.int32)
    loss = cf()
    dh = np.empty_like(h) if with_grads else None
    dw = np.empty_like(w) if with_grads else None
    if lib().qto_cross_entropy(h, h.shape[0], h.shape[1], w, w.shape[0], t, int(with_grads), C.byref(loss), dh,
                               dw) != 0:
        raise IndexError("cross entropy: target id out of range")
    return loss.value, dh, dw


def adamw_tensor(name, p, m, v, g, *, lr=1e-3, b1=0.9, b2=0.95, eps=1e-8, wd=0.0, bf16_moments=False,
                 bf16_params=True, seed=0, step_count=0, grad_scale=1.0, lo=0, hi=None):
    p, m, v, g = _f32(p).copy(), _f32(m).copy(), _f32(v).copy(), _f32(g)
    n = p.size
    hi = n if hi is None else hi
    rc = lib().qto_adamw_range(name.encode(), p, m, v, g, n, lo, hi, lr, b1, b2, eps, wd, int(bf16_moments),
                               int(bf16_params), seed, step_count + 1, grad_scale)
    if rc != 0:
        raise RuntimeError(f"adamw_step: non-finite gradient in {name}")
    return p, m, v


def grad_norm_partials(g, lo=0, hi=None) -> float:
    g = _f32(g).ravel()
    return lib().qto_grad_norm_partials(g, lo, g.size if hi is None else hi)


def grad_accumulate(name, buf, g, *, f32_mode=False, seed=0, micro_step=0):
    buf = _f32(buf).copy()
    lib().qto_grad_accumulate(name.encode(), buf, _f32(g), buf.size, int(f32_mode), seed, micro_step)
    return buf


def init_normal(n: int, std: float, seed: int, name: str) -> np.ndarray:
    out = np.empty(n, np.float32)
    lib().qto_init_normal(out, n, std, seed, name.encode())
    return out


def shard_layout(numel: int, workers: int) -> tuple[int, int]:
    a, b = i64(), i64()
    lib().qto_shard_layout(numel, workers, C.byref(a), C.byref(b))
    return a.value, b.value
