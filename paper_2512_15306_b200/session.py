"""Python mirror of the reference operator API (qtrain::ModelConfig,
PrecisionMap, RecomputeSet, RunPlan, AdamWHyper, model_forward/backward,
GradAccumulator, adamw_step / sharded_adamw_step, run_training's step) over
the native session in libqtrain_b200.so.

The reference is C++ (include/qtrain/model.hpp, include/qtrain/optim.hpp);
this module is the test/bench-facing host binding of the same entry points.
All compute runs on the GPU in the native library; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

# RecomputeSite bit order (include/qtrain/model.hpp:59)
RECOMPUTE_SITES = ("swiglu", "rmsnorm", "attention", "qkv", "ffn", "block")


def recompute_bits(names) -> int:
    """recompute_set_from_names (src/model.cpp:33-46)."""
    bits = 0
    for n in names or ():
        if n in ("none", ""):
            continue
        if n == "att":
            n = "attention"
        if n not in RECOMPUTE_SITES:
            raise ValueError(f"unknown recompute site: {n}")
        bits |= 1 << RECOMPUTE_SITES.index(n)
    return bits


# OffloadSet field order (include/qtrain/memplan.hpp:34-42) = QT_OFF_* bits
OFFLOAD_CATS = ("x", "m", "v", "master", "weights", "grads")
_OFFLOAD_ALIASES = {"residuals": "x", "theta*": "master", "theta": "weights", "g": "grads"}


def offload_bits(names) -> int:
    """offload_set_from_names (src/memplan.cpp:47-60)."""
    bits = 0
    for n in names or ():
        if n in ("none", ""):
            continue
        n = _OFFLOAD_ALIASES.get(n, n)
        if n not in OFFLOAD_CATS:
            raise ValueError(f"unknown offload category: {n}")
        bits |= 1 << OFFLOAD_CATS.index(n)
    return bits


@dataclass
class ModelConfig:
    n_layers: int = 2
    d_model: int = 64
    d_ff: int = 256
    n_heads: int = 4
    n_kv_heads: int = 2
    vocab: int = 512
    seq_len: int = 128

    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def qkv_dim(self) -> int:
        return self.d_model + 2 * self.n_kv_heads * self.head_dim()

    def as_list(self) -> list[int]:
        return [self.n_layers, self.d_model, self.d_ff, self.n_heads, self.n_kv_heads, self.vocab, self.seq_len]

    def block_linear_params(self) -> int:
        d, q, F = self.d_model, self.qkv_dim(), self.d_ff
        return self.n_layers * (q * d + d * d + F * d + d * (F // 2))

    def flops_per_token(self) -> tuple[float, float]:
        """(FP8, BF16) algorithmic FLOPs per token — flop_breakdown + mfu
        (src/memplan.cpp:264-312): 6 N_lin ; 6 V d + 12 (T/2) d L."""
        fp8 = 6.0 * self.block_linear_params()
        bf16 = 6.0 * self.vocab * self.d_model + 12.0 * (self.seq_len / 2.0) * self.d_model * self.n_layers
        return fp8, bf16


# model shapes named by BASELINE.json (src/memplan.cpp:93-106 presets; "tiny" and
# the Llama-7B shape are the survey's stated choices)
PRESETS = {
    "toy": ModelConfig(2, 64, 256, 4, 2, 512, 128),
    "tiny": ModelConfig(2, 256, 1536, 4, 4, 512, 256),
    "qwen2.5-0.5b": ModelConfig(24, 896, 9728, 14, 2, 151936, 1024),
    "qwen2.5-1.5b": ModelConfig(28, 1536, 17920, 12, 2, 151936, 1024),
    "llama-7b": ModelConfig(32, 4096, 22016, 32, 32, 32000, 1024),
    "qwen2.5-14b": ModelConfig(48, 5120, 27648, 40, 8, 152064, 1024),
}


@dataclass
class PrecisionMap:
    block_matmuls: str = "fp8"  # "fp8" | "bf16" (device path: fp8 only)
    backward_grads: str = "e4m3"  # "e4m3" | "e5m2"
    f32_debug: bool = False


@dataclass
class RunPlan:
    micro_batch: int = 1
    ga_steps: int = 1
    recompute: tuple = ()
    lmhead_chunk_tokens: int = 0
    attn_chunk_rows: int = 0
    shard_weights: bool = False
    shard_grads: bool = False
    moments: str = "f32"  # "f32" | "bf16_sr"
    offload: tuple = ()  # OffloadSet names (memplan.cpp:47-60): x, m, v, master, weights, grads
    transfer_policy: str = "double_buffer"  # "zero_copy" | "double_buffer"


@dataclass
class AdamWHyper:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0
    max_grad_norm: float = 1.0


class _Cfg(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("d_ff", C.c_int), ("n_heads", C.c_int),
                ("n_kv_heads", C.c_int), ("vocab", C.c_int64), ("seq_len", C.c_int)]


class _Prec(C.Structure):
    _fields_ = [("block_matmuls", C.c_int), ("backward_grads", C.c_int), ("f32_debug", C.c_int)]


class _Plan(C.Structure):
    _fields_ = [("micro_batch", C.c_int), ("ga_steps", C.c_int), ("recompute_bits", C.c_int),
                ("lmhead_chunk_tokens", C.c_int64), ("attn_chunk_rows", C.c_int64), ("shard_weights", C.c_int),
                ("shard_grads", C.c_int), ("bf16_moments", C.c_int), ("offload_bits", C.c_int),
                ("transfer_policy", C.c_int)]


class _Hyper(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("max_grad_norm", C.c_float)]


_vp, _i64, _u64, _ci = C.c_void_p, C.c_int64, C.c_uint64, C.c_int
_SIGS = {
    "qt_last_error": (C.c_char_p, []),
    "qt_nccl_unique_id": (_ci, [_vp]),
    "qt_session_create": (_ci, [C.POINTER(_Cfg), C.POINTER(_Prec), C.POINTER(_Plan), C.POINTER(_Hyper), _u64, _ci,
                                _ci, _vp, _ci, C.POINTER(_vp)]),
    "qt_session_destroy": (None, [_vp]),
    "qt_session_stream": (_vp, [_vp]),
    "qt_session_bytes": (C.c_size_t, [_vp]),
    "qt_num_params": (_ci, [_vp]),
    "qt_param_info": (_ci, [_vp, _ci, C.POINTER(C.c_char_p), C.POINTER(_i64)]),
    "qt_param_upload": (_ci, [_vp, _ci, _vp]),
    "qt_param_download": (_ci, [_vp, _ci, _vp]),
    "qt_grad_download": (_ci, [_vp, _ci, _vp]),
    "qt_reduced_grad_download": (_ci, [_vp, _ci, _vp]),
    "qt_moments_download": (_ci, [_vp, _ci, _vp, _vp]),
    "qt_moments_upload": (_ci, [_vp, _ci, _vp, _vp, _i64]),
    "qt_init_params": (_ci, [_vp, _u64]),
    "qt_build_step_context": (_ci, [_vp]),
    "qt_forward": (_ci, [_vp, _vp, _i64, _i64, _ci, _vp]),
    "qt_backward": (_ci, [_vp, _u64]),
    "qt_zero_grads": (_ci, [_vp]),
    "qt_grad_norm": (_ci, [_vp, C.POINTER(C.c_double)]),
    "qt_adamw_step": (_ci, [_vp, C.c_float]),
    "qt_train_step": (_ci, [_vp, _vp, _i64, _i64, _i64, C.c_float, _vp, _vp]),
    "qt_upload_tokens": (_ci, [_vp, _vp, _i64, C.POINTER(_vp)]),
    "qt_sync": (_ci, [_vp]),
    "qt_forward_stats": (_ci, [_vp, _vp]),
    "qt_saved_raw": (_ci, [_vp, _ci, C.c_char_p, _vp, C.POINTER(_i64), C.POINTER(_ci)]),
    "qt_scales": (_ci, [_vp, _ci, _vp]),
    "qt_weight_codes": (_ci, [_vp, _ci, _ci, _vp]),
    "qt_set_profile": (_ci, [_vp, _ci]),
    "qt_profile_read": (_ci, [_vp, _ci, _vp, _vp, _vp]),
    "qt_shard_layout": (_ci, [_i64, _ci, C.POINTER(_i64), C.POINTER(_i64)]),
    "qt_fnv1a64": (_u64, [C.c_char_p]),
    "qt_rope_table": (_ci, [_ci, _ci, _vp]),
    "qt_group_create": (_ci, [_ci, C.POINTER(_vp)]),
    "qt_group_destroy": (None, [_vp]),
    "qt_session_create_in_group": (_ci, [C.POINTER(_Cfg), C.POINTER(_Prec), C.POINTER(_Plan), C.POINTER(_Hyper),
                                         _u64, _vp, _ci, _ci, C.POINTER(_vp)]),
    "qt_session_transport": (C.c_char_p, [_vp]),
    "qt_count_step_kernels": (_ci, [_vp, _vp, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64)]),
}
_bound = False

# profile categories (session.cu prof_end ids)
PROFILE_CATS = ("gemm_fp8", "gemm_bf16", "unused", "quant", "rmsnorm", "elementwise", "attn_fwd", "ce_softmax",
                "attn_bwd", "comm", "adamw")


class QtError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def lib():
    global _bound
    l = _lib.lib()
    if not _bound:
        for n, (rt, at) in _SIGS.items():
            f = getattr(l, n)
            f.restype = rt
            f.argtypes = at
        _bound = True
    return l


def _chk(rc: int) -> None:
    if rc != 0:
        msg = lib().qt_last_error().decode()
        if rc == 1:
            raise ValueError(msg)  # std::invalid_argument
        if rc == 2:
            raise IndexError(msg)  # std::out_of_range
        raise QtError(rc, msg)  # std::runtime_error


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(lib().qt_nccl_unique_id(buf))
    return buf.raw


def shard_layout(numel: int, workers: int) -> tuple[int, int]:
    """shard_layout (src/comms.cpp:69-73) from the native library."""
    p, w = _i64(), _i64()
    _chk(lib().qt_shard_layout(numel, workers, C.byref(p), C.byref(w)))
    return p.value, w.value


def rope_table(T: int, hd: int) -> np.ndarray:
    """The session's RoPE table: (T, hd/2, 2) float32 {cos, sin}."""
    out = np.empty((T, hd // 2, 2), np.float32)
    _chk(lib().qt_rope_table(T, hd, out.ctypes.data))
    return out


def fnv1a64(s: str) -> int:
    return lib().qt_fnv1a64(s.encode())


class WorkerGroup:
    """In-process worker group (qtrain::WorkerGroup, include/qtrain/comms.hpp:51-78):
    `world` sessions driven by one host thread each, whose collectives are
    copy-engine pulls between the sessions' device arenas (qt_group_create)."""

    def __init__(self, world: int):
        out = _vp()
        _chk(lib().qt_group_create(world, C.byref(out)))
        self.h, self.world = out, world

    def run(self, fn, *args_per_rank):
        """WorkerGroup::run (src/comms.cpp:19-36): fn(rank, *args) on one thread per
        rank; returns the per-rank results, re-raises the first exception."""
        import threading
        res, errs = [None] * self.world, [None] * self.world

        def body(r):
            try:
                res[r] = fn(r, *[a[r] for a in args_per_rank])
            except BaseException as e:  # noqa: BLE001 - rethrown below, like the reference
                errs[r] = e

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        return res

    def close(self):
        if getattr(self, "h", None):
            lib().qt_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Session:
    """One GPU's training state: params, grads, optimizer state, activations."""

    def __init__(self, cfg: ModelConfig, prec: PrecisionMap | None = None, plan: RunPlan | None = None,
                 hyper: AdamWHyper | None = None, seed: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, device: int = 0, group: WorkerGroup | None = None):
        self.cfg, self.prec = cfg, prec or PrecisionMap()
        self.plan, self.hyper = plan or RunPlan(), hyper or AdamWHyper()
        self.seed, self.rank, self.world = seed, rank, world
        c = _Cfg(*cfg.as_list())
        p = _Prec(0 if self.prec.block_matmuls == "fp8" else 1, 0 if self.prec.backward_grads == "e4m3" else 1,
                  int(self.prec.f32_debug))
        pl = _Plan(self.plan.micro_batch, self.plan.ga_steps, recompute_bits(self.plan.recompute),
                   self.plan.lmhead_chunk_tokens, self.plan.attn_chunk_rows, int(self.plan.shard_weights),
                   int(self.plan.shard_grads), int(self.plan.moments == "bf16_sr"), offload_bits(self.plan.offload),
                   0 if self.plan.transfer_policy == "zero_copy" else 1)
        h = _Hyper(self.hyper.lr, self.hyper.beta1, self.hyper.beta2, self.hyper.eps, self.hyper.weight_decay,
                   self.hyper.max_grad_norm)
        out = _vp()
        if group is not None:
            self.world = world = group.world
            self._group = group  # the group outlives its sessions
            _chk(lib().qt_session_create_in_group(C.byref(c), C.byref(p), C.byref(pl), C.byref(h), seed, group.h,
                                                  rank, device, C.byref(out)))
        else:
            idb = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            _chk(lib().qt_session_create(C.byref(c), C.byref(p), C.byref(pl), C.byref(h), seed, rank, world, idb,
                                         device, C.byref(out)))
        self.h = out
        n = lib().qt_num_params(self.h)
        self.names, self.numel = [], []
        for i in range(n):
            nm, ne = C.c_char_p(), _i64()
            _chk(lib().qt_param_info(self.h, i, C.byref(nm), C.byref(ne)))
            self.names.append(nm.value.decode())
            self.numel.append(ne.value)

    def close(self):
        if getattr(self, "h", None):
            lib().qt_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().qt_session_stream(self.h)

    @property
    def transport(self) -> str:
        return lib().qt_session_transport(self.h).decode()

    @property
    def device_bytes(self) -> int:
        return lib().qt_session_bytes(self.h)

    # ---- parameters --------------------------------------------------------
    def _i(self, name: str) -> int:
        return self.names.index(name)

    def upload(self, name: str, values) -> None:
        v = np.ascontiguousarray(values, np.float32).ravel()
        i = self._i(name)
        if v.size != self.numel[i]:
            raise ValueError(f"{name}: expected {self.numel[i]} values, got {v.size}")
        _chk(lib().qt_param_upload(self.h, i, v.ctypes.data))

    def download(self, name: str) -> np.ndarray:
        i = self._i(name)
        out = np.empty(self.numel[i], np.float32)
        _chk(lib().qt_param_download(self.h, i, out.ctypes.data))
        return out

    def grad(self, name: str) -> np.ndarray:
        i = self._i(name)
        out = np.empty(self.numel[i], np.float32)
        _chk(lib().qt_grad_download(self.h, i, out.ctypes.data))
        return out

    def reduced_grad(self, name: str) -> np.ndarray:
        """world > 1: the cross-rank reduced f32 gradient (every rank's shard gathered)."""
        i = self._i(name)
        out = np.empty(self.numel[i], np.float32)
        _chk(lib().qt_reduced_grad_download(self.h, i, out.ctypes.data))
        return out

    def moments(self, name: str):
        """AdamW moments; with world > 1 this rank's ZeRO-1 slice [rank*pw, (rank+1)*pw)."""
        i = self._i(name)
        n = self.numel[i]
        m, v = np.empty(n, np.float32), np.empty(n, np.float32)
        _chk(lib().qt_moments_download(self.h, i, m.ctypes.data, v.ctypes.data))
        if self.world > 1:
            _, pw = shard_layout(n, self.world)
            k = max(0, min(pw, n - self.rank * pw))
            return m[:k], v[:k]
        return m, v

    def set_moments(self, name: str, m, v, step_count: int) -> None:
        m = np.ascontiguousarray(m, np.float32).ravel()
        v = np.ascontiguousarray(v, np.float32).ravel()
        _chk(lib().qt_moments_upload(self.h, self._i(name), m.ctypes.data, v.ctypes.data, step_count))

    def init_params(self, seed: int) -> None:
        _chk(lib().qt_init_params(self.h, seed))

    # ---- step pieces -------------------------------------------------------
    def build_step_context(self) -> None:
        _chk(lib().qt_build_step_context(self.h))

    def _tokens_dev(self, tokens):
        """tokens: a CUDA int32 tensor (device pointer used directly) or host
        array (staged through the session's token buffer)."""
        if hasattr(tokens, "data_ptr") and getattr(tokens, "is_cuda", False):
            return tokens.data_ptr(), tokens.numel()
        t = np.ascontiguousarray(tokens, np.int32).ravel()
        dev = _vp()
        _chk(lib().qt_upload_tokens(self.h, t.ctypes.data, t.size, C.byref(dev)))
        return dev.value, t.size

    def forward(self, tokens, batch: int, with_grads: bool = True, sync: bool = True):
        ptr, n = self._tokens_dev(tokens)
        loss = C.c_float()
        _chk(lib().qt_forward(self.h, ptr, n, batch, int(with_grads), C.byref(loss) if sync else None))
        return loss.value if sync else None

    def backward(self, micro_step: int) -> None:
        _chk(lib().qt_backward(self.h, micro_step))

    def zero_grads(self) -> None:
        _chk(lib().qt_zero_grads(self.h))

    def grad_norm(self) -> float:
        out = C.c_double()
        _chk(lib().qt_grad_norm(self.h, C.byref(out)))
        return out.value

    def adamw_step(self, grad_scale: float = 1.0) -> None:
        _chk(lib().qt_adamw_step(self.h, grad_scale))

    def train_step(self, tokens, batch: int, step: int, max_grad_norm: float | None = None, sync: bool = True):
        ptr, n = self._tokens_dev(tokens)
        per_mb = n // self.plan.ga_steps
        loss, norm = C.c_float(), C.c_float()
        mg = self.hyper.max_grad_norm if max_grad_norm is None else max_grad_norm
        _chk(lib().qt_train_step(self.h, ptr, per_mb, batch, step, mg, C.byref(loss) if sync else None,
                                 C.byref(norm) if sync else None))
        return (loss.value, norm.value) if sync else None

    def sync(self) -> None:
        _chk(lib().qt_sync(self.h))

    # ---- inspection ----------------------------------------------------------
    def forward_stats(self) -> np.ndarray:
        out = np.empty(self.cfg.n_layers * 4, np.uint32)
        _chk(lib().qt_forward_stats(self.h, out.ctypes.data))
        return out.view(np.float32).reshape(-1, 4)

    def saved(self, layer: int, site: str):
        nb, dt = _i64(), _ci()
        _chk(lib().qt_saved_raw(self.h, layer, site.encode(), None, C.byref(nb), C.byref(dt)))
        buf = np.empty(nb.value, np.uint8)
        _chk(lib().qt_saved_raw(self.h, layer, site.encode(), buf.ctypes.data, C.byref(nb), C.byref(dt)))
        if dt.value == 0:
            return (buf.view(np.uint16).astype(np.uint32) << 16).view(np.float32)
        if dt.value == 2:
            return buf.view(np.float32)
        return buf

    def scales(self, which: int) -> np.ndarray:
        out = np.empty(self.cfg.n_layers * 4, np.float32)
        _chk(lib().qt_scales(self.h, which, out.ctypes.data))
        return out.reshape(-1, 4)

    def weight_codes(self, layer: int, which: int) -> np.ndarray:
        c = self.cfg
        n = [c.qkv_dim() * c.d_model, c.d_model ** 2, c.d_ff * c.d_model, c.d_model * c.d_ff // 2][which]
        out = np.empty(n, np.uint8)
        _chk(lib().qt_weight_codes(self.h, layer, which, out.ctypes.data))
        return out

    def count_step_kernels(self, tokens, batch: int) -> tuple[int, int]:
        ptr, n = self._tokens_dev(tokens)
        k, o = _i64(), _i64()
        _chk(lib().qt_count_step_kernels(self.h, ptr, n // self.plan.ga_steps, batch, C.byref(k), C.byref(o)))
        return k.value, o.value

    def set_profile(self, on: bool) -> None:
        _chk(lib().qt_set_profile(self.h, int(on)))

    def profile(self) -> dict:
        n = len(PROFILE_CATS)
        ms, ln, wk = np.zeros(n), np.zeros(n, np.int64), np.zeros(n)
        _chk(lib().qt_profile_read(self.h, n, ms.ctypes.data, ln.ctypes.data, wk.ctypes.data))
        return {c: {"ms": float(ms[i]), "launches": int(ln[i]), "work": float(wk[i])}
                for i, c in enumerate(PROFILE_CATS) if ln[i]}
