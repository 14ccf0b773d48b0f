"""ctypes binding of the native library (libqtrain_b200.so, built in-tree).

There is no fallback: if the library is missing or a CUDA device is absent the
caller gets an exception, never a CPU emulation.
"""
from __future__ import annotations

import ctypes as C
import pathlib

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libqtrain_b200.so"

c_i64 = C.c_int64
c_u64 = C.c_uint64
c_vp = C.c_void_p


class QtkGemm(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("a_fmt", C.c_int), ("b_fmt", C.c_int), ("a_mn", C.c_int), ("b_mn", C.c_int),
        ("M", c_i64), ("N", c_i64), ("K", c_i64),
        ("a", c_vp), ("lda", c_i64), ("b", c_vp), ("ldb", c_i64),
        ("a_scale", c_vp), ("b_scale", c_vp),
        ("epi", C.c_int), ("out", c_vp), ("ldo", c_i64), ("res", c_vp), ("ldr", c_i64),
        ("sr_seed", c_u64), ("sr_stream", c_u64), ("sr_base", c_u64), ("bn", C.c_int), ("a2", c_vp),
        ("ws", c_vp), ("ws_bytes", c_i64), ("split_k", C.c_int), ("amax", c_vp),
        ("ce_targets", c_vp), ("ce_stats", c_vp), ("ce_tgt_logit", c_vp), ("sr_micro_step", c_vp),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "qtk_absmax_bf16": (C.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "qtk_absmax_f32": (C.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "qtk_quantize_bf16": (C.c_int, [c_vp, c_i64, C.c_int, c_vp, c_vp, c_vp, c_vp]),
    "qtk_quantize_transpose_bf16": (C.c_int, [c_vp, c_i64, c_i64, C.c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "qtk_gemm": (C.c_int, [C.POINTER(QtkGemm), c_vp]),
    "qtk_gemm_splitk_ws_bytes": (C.c_int, [c_i64, c_i64, c_i64, C.c_int]),
    "qtk_ce_softmax": (C.c_int, [c_vp, c_i64, c_i64, C.c_int, c_vp, C.c_float, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "qtk_reduce_scatter_sr": (C.c_int, [c_vp, C.POINTER(c_vp), C.c_int, C.c_int, c_i64, C.c_int, c_u64, c_u64, c_u64,
                                        c_vp]),
    "qt_time_graph_step": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, C.c_int, C.POINTER(C.c_float)]),
    "qtk_ce_softmax_stats": (C.c_int, [c_vp, c_i64, c_i64, C.c_int, c_vp, c_vp, c_vp, C.c_float, c_vp, c_vp, c_i64, c_vp,
                                       c_vp]),
    "qtk_ce_softmax_stats_tx": (C.c_int, [c_vp, c_i64, c_i64, C.c_int, c_vp, c_vp, c_vp, C.c_float, c_vp, c_i64, c_vp,
                                          c_vp, c_vp]),
    "qtk_lm_dgrad_finish": (C.c_int, [c_vp, c_i64, C.c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "qtk_lm_wgrad_targets": (C.c_int, [c_vp, C.c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "qtk_attn_fwd": (C.c_int, [c_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, c_vp, c_i64, c_vp, c_vp,
                               c_vp, c_vp]),
    "qtk_attn_bwd": (C.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_int, c_vp, c_vp, c_vp]),
    "qtk_attn_bwd_ws_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "qtk_rmsnorm_fwd": (C.c_int, [c_vp, c_vp, c_vp, c_i64, C.c_int, C.c_float, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "qtk_rmsnorm_bwd": (C.c_int, [c_vp, c_vp, c_i64, C.c_int, C.c_float, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "qtk_rmsnorm_bwd_partials": (C.c_int, [c_i64, C.c_int]),
    "qtk_swiglu_fwd": (C.c_int, [c_vp, c_i64, C.c_int, c_vp, c_vp, c_vp]),
    "qtk_swiglu_bwd": (C.c_int, [c_vp, c_vp, c_i64, C.c_int, c_vp, c_vp, c_vp]),
    "qtk_swiglu_selfcheck": (C.c_int, [c_vp, c_vp]),
    "qtk_attn_set_mode": (None, [C.c_int, C.c_int]),
    "qtk_attn_set_plo": (None, [C.c_int]),
    "qtk_attn_set_fwd2q": (None, [C.c_int]),
    "qtk_rms_set_path": (None, [C.c_int]),
    "qtk_rope_set_heads": (None, [C.c_int]),
    "qtk_rope": (C.c_int, [c_vp, c_i64, C.c_int, C.c_int, C.c_int, C.c_int, c_vp, C.c_int, c_vp, c_vp]),
    "qtk_gemm_plan": (C.c_int, [C.POINTER(QtkGemm)] + [C.POINTER(C.c_int)] * 5),
    "qtk_gemm_tail_plan": (C.c_int, [C.POINTER(QtkGemm), C.POINTER(c_i64), C.POINTER(C.c_int)]),
    "qtk_embed_fwd": (C.c_int, [c_vp, C.c_int, C.c_int, c_vp, C.c_int, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "qtk_embed_sort_scratch_bytes": (C.c_size_t, [C.c_int, c_i64]),
    "qtk_embed_sort": (C.c_int, [c_vp, C.c_int, c_i64, c_vp, C.c_size_t, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "qtk_embed_bwd": (C.c_int, [c_vp, c_vp, c_vp, c_vp, C.c_int, c_vp, C.c_int, c_vp, c_u64, c_u64, c_u64, c_vp]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2512_15306_b200.build` "
                               "(there is no CPU fallback)")
        l = C.CDLL(str(LIB_PATH))
        for name, (rt, at) in _SIGS.items():
            f = getattr(l, name)
            f.restype = rt
            f.argtypes = at
        _lib = l
    return _lib


def declared_symbols() -> list[str]:
    return sorted(_SIGS)


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = ""
        try:
            f = lib().qt_last_error
            f.restype = C.c_char_p
            msg = (f() or b"").decode()
        except AttributeError:
            pass
        raise RuntimeError(f"{what} failed with status {rc} {msg}")
