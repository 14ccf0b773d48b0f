"""ctypes/numpy binding of oracle/_ref/libqtrain_ref.so — the UNMODIFIED
reference (qtrain) compiled from /root/reference/proj/src by oracle/Makefile.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, always as the checker or the
timed CPU baseline, never on the product path.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libqtrain_ref.so"

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64, u64, ci, cf, vp = C.c_int64, C.c_uint64, C.c_int, C.c_float, C.c_void_p


class _OptF32(object):
    """ndpointer that also accepts None."""

    @classmethod
    def from_param(cls, obj):
        if obj is None:
            return None
        return f32p.from_param(obj)


_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_f8_encode": (ci, [f32p, i64, ci, u8p]),
    "ref_f8_decode_table": (ci, [ci, f32p]),
    "ref_f8_fmax": (cf, [ci]),
    "ref_absmax": (ci, [f32p, i64, C.POINTER(cf)]),
    "ref_absmax_scale": (cf, [cf, ci]),
    "ref_quantize_with_absmax": (ci, [f32p, i64, ci, cf, u8p, C.POINTER(cf)]),
    "ref_transpose_quantize_with_absmax": (ci, [f32p, i64, i64, ci, cf, u8p, C.POINTER(cf)]),
    "ref_rng_uniform": (C.c_uint32, [u64, u64, u64]),
    "ref_rng_normal": (cf, [u64, u64, u64]),
    "ref_fnv1a64": (u64, [C.c_char_p]),
    "ref_bf16_round": (cf, [cf]),
    "ref_stochastic_round_bf16": (cf, [cf, u64, u64, u64]),
    "ref_matmul_fp8": (ci, [u8p, i64, i64, ci, cf, u8p, i64, ci, cf, ci, f32p]),
    "ref_matmul_f32": (ci, [f32p, i64, i64, f32p, i64, ci, f32p]),
    "ref_rmsnorm_residual_fused": (ci, [_OptF32, f32p, f32p, i64, i64, cf, f32p, f32p, C.POINTER(cf)]),
    "ref_rmsnorm_residual_backward": (ci, [f32p, f32p, i64, i64, cf, f32p, _OptF32, f32p, f32p]),
    "ref_swiglu_fused": (ci, [f32p, i64, i64, f32p, C.POINTER(cf)]),
    "ref_swiglu_backward": (ci, [f32p, i64, i64, f32p, f32p]),
    "ref_sdpa": (ci, [f32p, f32p, f32p, i64, i64, i64, i64, i64, f32p]),
    "ref_sdpa_backward": (ci, [f32p, f32p, f32p, f32p, i64, i64, i64, i64, i64, f32p, f32p, f32p]),
    "ref_embedding_backward": (ci, [i32p, i64, f32p, i64, i64, f32p]),
    "ref_cross_entropy": (ci, [f32p, i64, i64, f32p, i64, i32p, i64, ci, C.POINTER(cf), _OptF32, _OptF32]),
    "ref_adamw_tensor": (ci, [C.c_char_p, f32p, f32p, f32p, f32p, i64, cf, cf, cf, cf, cf, ci, ci, u64, i64, cf]),
    "ref_grad_norm_partials": (C.c_double, [f32p, i64]),
    "ref_grad_accumulate": (ci, [C.c_char_p, f32p, f32p, i64, ci, u64, u64]),
    "ref_model_new": (vp, [C.POINTER(ci), u64, ci, ci, ci]),
    "ref_model_free": (None, [vp]),
    "ref_model_set_options": (ci, [vp, ci, i64, i64, cf, cf, cf, cf, cf, ci]),
    "ref_model_num_params": (ci, [vp]),
    "ref_model_param_name": (C.c_char_p, [vp, ci]),
    "ref_model_param_numel": (i64, [vp, ci]),
    "ref_model_get_param": (None, [vp, ci, f32p]),
    "ref_model_set_param": (None, [vp, ci, f32p]),
    "ref_model_get_moments": (ci, [vp, ci, f32p, f32p]),
    "ref_model_set_moments": (ci, [vp, ci, f32p, f32p, i64]),
    "ref_model_fwd_bwd": (ci, [vp, i32p, i64, i64, ci, C.POINTER(cf)]),
    "ref_model_forward_stats": (None, [vp, f32p]),
    "ref_model_saved": (i64, [vp, ci, C.c_char_p, _OptF32]),
    "ref_model_grad": (ci, [vp, C.c_char_p, f32p]),
    "ref_model_acc_grad": (ci, [vp, C.c_char_p, f32p]),
    "ref_model_train_step": (ci, [vp, i32p, i64, i64, ci, ci, i64, cf, C.POINTER(cf), C.POINTER(cf)]),
    "ref_model_time_step": (C.c_double, [vp, i32p, i64, i64, i64]),
    "ref_make_corpus": (ci, [ci, i64, ci, ci, ci, u64, i32p, i32p]),
    "ref_flops_per_token": (None, [C.POINTER(ci), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "ref_reduce_scatter_oracle": (ci, [f32p, f32p, ci, i64, ci, u64, u64, u64]),
    "ref_reduce_scatter_copy": (ci, [f32p, f32p, ci, i64, ci, u64, u64, u64]),
    "ref_rope_apply": (ci, [C.POINTER(ci), f32p, i64, i64, ci]),
    "ref_memory_breakdown": (ci, [C.POINTER(ci), ci, C.POINTER(i64), ci, C.POINTER(u64)]),
    "ref_flop_breakdown": (ci, [C.POINTER(ci), ci, ci, C.POINTER(C.c_double)]),
    "ref_mfu": (ci, [C.c_double, C.POINTER(ci), ci, C.c_char_p, ci, C.POINTER(C.c_double)]),
    "ref_fp8_speedup_ceiling": (ci, [C.POINTER(ci), C.c_char_p, ci, C.POINTER(C.c_double)]),
    "ref_estimate_step_time": (ci, [C.POINTER(ci), C.POINTER(i64), C.c_char_p, ci, ci, C.POINTER(C.c_double)]),
    "ref_search_plan": (ci, [C.POINTER(ci), C.c_char_p, ci, i64, ci, ci, ci, C.c_char_p, C.c_size_t]),
    "ref_plan_residency": (ci, [C.POINTER(ci), C.POINTER(i64), u64, ci, C.c_char_p, C.c_size_t]),
    "ref_profile_json": (ci, [C.c_char_p, C.c_char_p, C.c_size_t]),
    "ref_transfer_time": (ci, [u64, C.c_char_p, ci, C.POINTER(C.c_double)]),
    "ref_manifest_normalize": (ci, [C.c_char_p, C.c_char_p, C.c_size_t]),
    "ref_run_training": (ci, [C.c_char_p, C.c_char_p, C.c_size_t]),
}

_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} not built (make -C oracle ref; needs /root/reference)")
        l = C.CDLL(str(REF_LIB))
        for n, (rt, at) in _SIGS.items():
            f = getattr(l, n)
            f.restype = rt
            f.argtypes = at
        _lib = l
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _chk(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ---- numerics -------------------------------------------------------------
def f8_encode(x, kind: int) -> np.ndarray:
    x = _f32(x).ravel()
    out = np.empty(x.size, np.uint8)
    _chk(lib().ref_f8_encode(x, x.size, kind, out))
    return out


def f8_decode_table(kind: int) -> np.ndarray:
    out = np.empty(256, np.float32)
    _chk(lib().ref_f8_decode_table(kind, out))
    return out


def absmax(x) -> float:
    x = _f32(x).ravel()
    r = cf()
    _chk(lib().ref_absmax(x, x.size, C.byref(r)))
    return r.value


def absmax_scale(a: float, kind: int) -> float:
    return lib().ref_absmax_scale(a, kind)


def quantize_with_absmax(x, kind: int, amax: float) -> tuple[np.ndarray, float]:
    x = _f32(x)
    codes = np.empty(x.size, np.uint8)
    s = cf()
    _chk(lib().ref_quantize_with_absmax(x.ravel(), x.size, kind, amax, codes, C.byref(s)))
    return codes.reshape(x.shape), s.value


def transpose_quantize_with_absmax(x, kind: int, amax: float) -> tuple[np.ndarray, float]:
    x = _f32(x)
    r, c = x.shape
    codes = np.empty(r * c, np.uint8)
    s = cf()
    _chk(lib().ref_transpose_quantize_with_absmax(x, r, c, kind, amax, codes, C.byref(s)))
    return codes.reshape(c, r), s.value


def rng_uniform(seed: int, stream: int, counter: int) -> int:
    return lib().ref_rng_uniform(seed, stream, counter)


def fnv1a64(s: str) -> int:
    return lib().ref_fnv1a64(s.encode())


def bf16_round(x: float) -> float:
    return lib().ref_bf16_round(x)


def stochastic_round_bf16(x: float, seed: int, stream: int, counter: int) -> float:
    return lib().ref_stochastic_round_bf16(x, seed, stream, counter)


# ---- tensorops ------------------------------------------------------------
def matmul_fp8(a_codes, a_kind, a_scale, b_codes, b_kind, b_scale, round_bf16=True) -> np.ndarray:
    a = np.ascontiguousarray(a_codes, np.uint8)
    b = np.ascontiguousarray(b_codes, np.uint8)
    M, K = a.shape
    N = b.shape[0]
    out = np.empty((M, N), np.float32)
    _chk(lib().ref_matmul_fp8(a, M, K, a_kind, a_scale, b, N, b_kind, b_scale, int(round_bf16), out))
    return out


def matmul_f32(a, b, round_bf16=True) -> np.ndarray:
    a, b = _f32(a), _f32(b)
    out = np.empty((a.shape[0], b.shape[0]), np.float32)
    _chk(lib().ref_matmul_f32(a, a.shape[0], a.shape[1], b, b.shape[0], int(round_bf16), out))
    return out


def rmsnorm_residual_fused(x, res, gamma, eps=1e-6):
    res, gamma = _f32(res), _f32(gamma)
    rows, d = res.shape
    nr = np.empty_like(res)
    normed = np.empty_like(res)
    am = cf()
    _chk(lib().ref_rmsnorm_residual_fused(None if x is None else _f32(x), res, gamma, rows, d, eps, nr, normed,
                                          C.byref(am)))
    return nr, normed, am.value


def rmsnorm_residual_backward(nr, gamma, dy, d_extra=None, eps=1e-6):
    nr, gamma, dy = _f32(nr), _f32(gamma), _f32(dy)
    rows, d = nr.shape
    din = np.empty_like(nr)
    dg = np.empty(d, np.float32)
    _chk(lib().ref_rmsnorm_residual_backward(nr, gamma, rows, d, eps, dy,
                                             None if d_extra is None else _f32(d_extra), din, dg))
    return din, dg


def swiglu_fused(gu):
    gu = _f32(gu)
    rows, two_h = gu.shape
    h = np.empty((rows, two_h // 2), np.float32)
    am = cf()
    _chk(lib().ref_swiglu_fused(gu, rows, two_h, h, C.byref(am)))
    return h, am.value


def swiglu_backward(gu, dh):
    gu, dh = _f32(gu), _f32(dh)
    out = np.empty_like(gu)
    _chk(lib().ref_swiglu_backward(gu, gu.shape[0], gu.shape[1], dh, out))
    return out


def sdpa(q, k, v, chunk_rows=0):
    q, k, v = _f32(q), _f32(k), _f32(v)
    H, T, D = q.shape
    out = np.empty_like(q)
    _chk(lib().ref_sdpa(q, k, v, H, k.shape[0], T, D, chunk_rows or T, out))
    return out


def sdpa_backward(q, k, v, go, chunk_rows=0):
    q, k, v, go = _f32(q), _f32(k), _f32(v), _f32(go)
    H, T, D = q.shape
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    _chk(lib().ref_sdpa_backward(q, k, v, go, H, k.shape[0], T, D, chunk_rows or T, dq, dk, dv))
    return dq, dk, dv


def rope_apply(cfg7, qkv, batch: int, seq: int, backward: bool = False) -> np.ndarray:
    """The reference's own rope_apply (src/model.cpp:169-191, internal to
    model.cpp; exported by oracle/ref_internal.cpp) on a (batch*seq, qkv_dim)
    f32 tensor; returns the rotated copy."""
    x = _f32(qkv).copy()
    arr = (ci * 7)(*cfg7)
    _chk(lib().ref_rope_apply(arr, x, batch, seq, int(backward)))
    return x


def embedding_backward(ids, grad_out, vocab):
    ids = np.ascontiguousarray(ids, np.int32)
    g = _f32(grad_out)
    out = np.empty((vocab, g.shape[1]), np.float32)
    _chk(lib().ref_embedding_backward(ids, ids.size, g, g.shape[1], vocab, out))
    return out


def cross_entropy(hidden, lm_w, targets, chunk=0, with_grads=True):
    h, w = _f32(hidden), _f32(lm_w)
    t = np.ascontiguousarray(targets, np.int32)
    N, d = h.shape
    V = w.shape[0]
    loss = cf()
    dh = np.empty_like(h) if with_grads else None
    dw = np.empty_like(w) if with_grads else None
    _chk(lib().ref_cross_entropy(h, N, d, w, V, t, chunk or N, int(with_grads), C.byref(loss), dh, dw))
    return loss.value, dh, dw


# ---- optimizer --------------------------------------------------------------
def adamw_tensor(name, p, m, v, g, *, lr=1e-3, b1=0.9, b2=0.95, eps=1e-8, wd=0.0, bf16_moments=False,
                 bf16_params=True, seed=0, step_count=0, grad_scale=1.0):
    p, m, v, g = _f32(p).copy(), _f32(m).copy(), _f32(v).copy(), _f32(g)
    _chk(lib().ref_adamw_tensor(name.encode(), p, m, v, g, p.size, lr, b1, b2, eps, wd, int(bf16_moments),
                                int(bf16_params), seed, step_count, grad_scale))
    return p, m, v


def grad_norm_partials(g) -> float:
    g = _f32(g).ravel()
    return lib().ref_grad_norm_partials(g, g.size)


def grad_accumulate(name, buf, g, *, f32_mode=False, seed=0, micro_step=0):
    buf = _f32(buf).copy()
    _chk(lib().ref_grad_accumulate(name.encode(), buf, _f32(g), buf.size, int(f32_mode), seed, micro_step))
    return buf


def make_corpus(kind: str, vocab: int, seq_len: int, n_train: int, n_val: int, seed: int):
    tr = np.empty(n_train * (seq_len + 1), np.int32)
    va = np.empty(max(n_val, 0) * (seq_len + 1), np.int32)
    _chk(lib().ref_make_corpus(int(kind == "uniform"), vocab, seq_len, n_train, n_val, seed, tr, va))
    return tr, va


def flops_per_token(cfg7) -> tuple[float, float]:
    arr = (ci * 7)(*cfg7)
    a, b = C.c_double(), C.c_double()
    lib().ref_flops_per_token(arr, C.byref(a), C.byref(b))
    return a.value, b.value


# ---- model handle -------------------------------------------------------------
class RefModel:
    """The reference model + optimizer state (src/model.cpp, src/optim.cpp,
    src/trainer.cpp:64-131) behind a handle."""

    SITES = ("r_in", "n1", "qkv", "att", "r_mid", "n2", "gate_up", "h")

    def __init__(self, cfg7, seed: int, *, fp8=True, grad_e5m2=False, f32_debug=False, recompute_bits=0,
                 lmhead_chunk=0, attn_chunk=0, lr=1e-3, b1=0.9, b2=0.95, eps=1e-8, wd=0.0, bf16_moments=False):
        self.cfg7 = list(cfg7)
        arr = (ci * 7)(*cfg7)
        h = lib().ref_model_new(arr, seed, 0 if fp8 else 1, 1 if grad_e5m2 else 0, int(f32_debug))
        if not h:
            raise RefError(1, lib().ref_last_error().decode())
        self.h = h
        _chk(lib().ref_model_set_options(h, recompute_bits, lmhead_chunk, attn_chunk, lr, b1, b2, eps, wd,
                                         int(bf16_moments)))
        n = lib().ref_model_num_params(h)
        self.names = [lib().ref_model_param_name(h, i).decode() for i in range(n)]
        self.numel = [lib().ref_model_param_numel(h, i) for i in range(n)]

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_model_free(self.h)
            self.h = None

    def get(self, name: str) -> np.ndarray:
        i = self.names.index(name)
        out = np.empty(self.numel[i], np.float32)
        lib().ref_model_get_param(self.h, i, out)
        return out

    def set(self, name: str, val) -> None:
        i = self.names.index(name)
        v = _f32(val).ravel()
        assert v.size == self.numel[i]
        lib().ref_model_set_param(self.h, i, v)

    def params(self) -> dict[str, np.ndarray]:
        return {n: self.get(n) for n in self.names}

    def moments(self, name: str):
        i = self.names.index(name)
        m = np.empty(self.numel[i], np.float32)
        v = np.empty(self.numel[i], np.float32)
        _chk(lib().ref_model_get_moments(self.h, i, m, v))
        return m, v

    def set_moments(self, name: str, m, v, step_count: int) -> None:
        i = self.names.index(name)
        _chk(lib().ref_model_set_moments(self.h, i, _f32(m).ravel(), _f32(v).ravel(), step_count))

    def fwd_bwd(self, tokens, batch: int, with_grads: bool = True) -> float:
        t = np.ascontiguousarray(tokens, np.int32)
        loss = cf()
        _chk(lib().ref_model_fwd_bwd(self.h, t, t.size, batch, int(with_grads), C.byref(loss)))
        return loss.value

    def stats(self) -> np.ndarray:
        out = np.empty(self.cfg7[0] * 4, np.float32)
        lib().ref_model_forward_stats(self.h, out)
        return out.reshape(-1, 4)

    def saved(self, layer: int, site: str):
        n = lib().ref_model_saved(self.h, layer, site.encode(), None)
        if n < 0:
            return None
        out = np.empty(n, np.float32)
        lib().ref_model_saved(self.h, layer, site.encode(), out)
        return out

    def grad(self, name: str) -> np.ndarray:
        i = self.names.index(name)
        out = np.empty(self.numel[i], np.float32)
        _chk(lib().ref_model_grad(self.h, name.encode(), out))
        return out

    def acc_grad(self, name: str) -> np.ndarray:
        i = self.names.index(name)
        out = np.empty(self.numel[i], np.float32)
        _chk(lib().ref_model_acc_grad(self.h, name.encode(), out))
        return out

    def train_step(self, tokens, batch: int, *, ga_steps=1, workers=1, step=0, max_grad_norm=1.0):
        t = np.ascontiguousarray(tokens, np.int32).ravel()
        per_mb = t.size // (ga_steps * workers)
        loss, norm = cf(), cf()
        _chk(lib().ref_model_train_step(self.h, t, per_mb, batch, ga_steps, workers, step, max_grad_norm,
                                        C.byref(loss), C.byref(norm)))
        return loss.value, norm.value

    def time_step(self, tokens, batch: int, step: int = 0) -> float:
        t = np.ascontiguousarray(tokens, np.int32).ravel()
        return lib().ref_model_time_step(self.h, t, t.size, batch, step)


def reduce_scatter(chunks, acc, *, stochastic=True, seed=0, step=0, layer=0, protocol=False):
    """reduce_scatter_oracle (or the copy protocol) of src/comms.cpp:185-254.
    chunks: (W, W, n) -- chunks[i][j] is worker i's chunk for shard j; acc: (W, n)."""
    c = np.ascontiguousarray(chunks, np.float32)
    a = np.ascontiguousarray(acc, np.float32).copy()
    W, n = a.shape
    f = lib().ref_reduce_scatter_copy if protocol else lib().ref_reduce_scatter_oracle
    _chk(f(c.ravel(), a.ravel(), W, n, int(stochastic), seed, step, layer))
    return a


# ---------------------------------------------------------------- planner (src/memplan.cpp, profiles.cpp, offload.cpp)
def _cfg7(cfg7):
    return (ci * 7)(*cfg7)


def _plan10(mb=1, ga=1, recompute_bits=0, offload_bits=0, shard_weights=False, shard_grads=False, bf16=False,
            bf16_moments=True, lmhead_chunk=512, attn_chunk=256):
    return (i64 * 10)(mb, ga, recompute_bits, offload_bits, int(shard_weights), int(shard_grads), int(bf16),
                      int(bf16_moments), lmhead_chunk, attn_chunk)


TIER = ("params_fp8", "params_bf16_master", "moments_m", "moments_v", "grads", "residuals", "activations",
        "logits_workspace", "attn_workspace")


def memory_breakdown(cfg7, workers=1, tied=False, **plan):
    out = (u64 * 18)()
    _chk(lib().ref_memory_breakdown(_cfg7(cfg7), int(tied), _plan10(**plan), workers, out))
    return dict(zip(TIER, out[:9])), dict(zip(TIER, out[9:]))


def flop_breakdown(cfg7, recompute_bits=0, tied=False):
    out = (C.c_double * 4)()
    _chk(lib().ref_flop_breakdown(_cfg7(cfg7), recompute_bits, int(tied), out))
    return dict(zip(("linear", "lmhead", "attention", "recompute"), out))


def mfu(tps, cfg7, profile, bf16=False, tied=False):
    out = C.c_double()
    _chk(lib().ref_mfu(tps, _cfg7(cfg7), int(bf16), profile.encode(), int(tied), C.byref(out)))
    return out.value


def fp8_speedup_ceiling(cfg7, profile, tied=False):
    out = C.c_double()
    _chk(lib().ref_fp8_speedup_ceiling(_cfg7(cfg7), profile.encode(), int(tied), C.byref(out)))
    return out.value


def estimate_step_time(cfg7, profile, workers=1, tied=False, **plan):
    out = (C.c_double * 7)()
    _chk(lib().ref_estimate_step_time(_cfg7(cfg7), _plan10(**plan), profile.encode(), workers, int(tied), out))
    return dict(zip(("compute", "transfer", "exposed_transfer", "optimizer", "total", "feasible_in_time",
                     "tokens_per_second"), out))


_SEARCH_CHILD = r"""
import ctypes as C, sys
l = C.CDLL(sys.argv[1])
f = l.ref_search_plan
f.argtypes = [C.POINTER(C.c_int), C.c_char_p, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
a = [int(x) for x in sys.argv[3:]]
buf = C.create_string_buffer(256 << 20)
rc = f((C.c_int * 7)(*a[:7]), sys.argv[2].encode(), *a[7:], buf, len(buf))
if rc:
    l.ref_last_error.restype = C.c_char_p
    sys.stderr.write(l.ref_last_error().decode())
    sys.exit(rc)
sys.stdout.write(buf.value.decode())
"""


def search_plan(cfg7, profile, workers, target, bf16=False, exhaustive=False, tied=False):
    """search_plan runs in a child interpreter that has not imported numpy: in a
    process where numpy (OpenBLAS) is loaded the reference's search_plan
    segfaults inside its std::sort (reproduced with the unmodified sources;
    the same call from C++ or from a numpy-free interpreter is fine)."""
    import json
    import subprocess
    import sys
    args = [str(x) for x in (*cfg7, workers, target, int(bf16), int(exhaustive), int(tied))]
    r = subprocess.run([sys.executable, "-c", _SEARCH_CHILD, str(REF_LIB), profile, *args], capture_output=True,
                       text=True, timeout=600)
    if r.returncode:
        raise RefError(r.returncode, r.stderr)
    return json.loads(r.stdout)


_RESIDENCY_CHILD = r"""
import ctypes as C, sys
l = C.CDLL(sys.argv[1])
f = l.ref_plan_residency
f.argtypes = [C.POINTER(C.c_int), C.POINTER(C.c_int64), C.c_uint64, C.c_int, C.c_char_p, C.c_size_t]
a = [int(x) for x in sys.argv[2:]]
buf = C.create_string_buffer(64 << 20)
rc = f((C.c_int * 7)(*a[:7]), (C.c_int64 * 10)(*a[7:17]), a[17], a[18], buf, len(buf))
if rc:
    l.ref_last_error.restype = C.c_char_p
    sys.stderr.write(l.ref_last_error().decode())
    sys.exit(rc)
sys.stdout.write(buf.value.decode())
"""


def plan_residency(cfg7, budget, tied=False, **plan):
    """Child interpreter for the same reason as search_plan (std::ostringstream
    inside the reference crashes once numpy/torch are loaded in this process)."""
    import json
    import subprocess
    import sys
    args = [str(int(x)) for x in (*cfg7, *_plan10(**plan), budget, int(tied))]
    r = subprocess.run([sys.executable, "-c", _RESIDENCY_CHILD, str(REF_LIB), *args], capture_output=True, text=True,
                       timeout=600)
    if r.returncode:
        raise RefError(r.returncode, r.stderr)
    return json.loads(r.stdout)


def profile_json(name):
    import json
    buf = C.create_string_buffer(1 << 16)
    _chk(lib().ref_profile_json(name.encode(), buf, len(buf)))
    return json.loads(buf.value.decode())


def transfer_time(nbytes, profile, zero_copy):
    out = C.c_double()
    _chk(lib().ref_transfer_time(nbytes, profile.encode(), 0 if zero_copy else 1, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- manifest / trainer (src/manifest.cpp, trainer.cpp)
def manifest_normalize(text: str) -> dict:
    import json
    buf = C.create_string_buffer(1 << 20)
    _chk(lib().ref_manifest_normalize(text.encode(), buf, len(buf)))
    return json.loads(buf.value.decode())


def run_training(manifest_text: str) -> str:
    """The reference trainer (run_training_to_files): writes the manifest's metrics CSV and
    checkpoint, returns the CSV text."""
    buf = C.create_string_buffer(16 << 20)
    _chk(lib().ref_run_training(manifest_text.encode(), buf, len(buf)))
    return buf.value.decode()
