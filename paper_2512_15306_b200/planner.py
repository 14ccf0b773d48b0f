"""Python mirror of the planner C ABI (csrc/planner.cpp; include/qtrain_b200.h).

Same names and meaning as the reference's planner (include/qtrain/memplan.hpp,
profiles.hpp, offload.hpp): memory_breakdown, flop_breakdown, mfu,
estimate_step_time, search_plan, plan_residency, transfer_time, and the
hardware profiles (builtins + "b200").  Host-only: none of these touch a GPU.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

from . import session as S

_vp, _i64, _u64, _ci = C.c_void_p, C.c_int64, C.c_uint64, C.c_int


class HardwareProfile(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("device_bytes", _u64), ("host_bytes", _u64),
                ("peak_flops_fp8", C.c_double), ("peak_flops_bf16", C.c_double), ("peak_flops_f32", C.c_double),
                ("mem_bandwidth", C.c_double), ("link_bandwidth", C.c_double), ("p2p", _ci),
                ("attainable_fraction", C.c_double), ("zero_copy_efficiency", C.c_double),
                ("double_buffer_efficiency", C.c_double)]


TIER_FIELDS = ("params_fp8", "params_bf16_master", "moments_m", "moments_v", "grads", "residuals", "activations",
               "logits_workspace", "attn_workspace")


class _Tier(C.Structure):
    _fields_ = [(f, _u64) for f in TIER_FIELDS]


class _Flops(C.Structure):
    _fields_ = [("linear", C.c_double), ("lmhead", C.c_double), ("attention", C.c_double),
                ("recompute", C.c_double)]


class _Time(C.Structure):
    _fields_ = [("compute", C.c_double), ("transfer", C.c_double), ("exposed_transfer", C.c_double),
                ("optimizer", C.c_double), ("total", C.c_double), ("feasible_in_time", _ci),
                ("tokens_per_second", C.c_double)]


_P = C.POINTER
_SIGS = {
    "qt_plan_last_error": (C.c_char_p, []),
    "qt_profile_by_name": (_ci, [C.c_char_p, _P(HardwareProfile)]),
    "qt_profile_load": (_ci, [C.c_char_p, _P(HardwareProfile)]),
    "qt_profile_from_json": (_ci, [C.c_char_p, _P(HardwareProfile)]),
    "qt_profile_to_json": (_ci, [_P(HardwareProfile), _vp, C.c_size_t, _P(C.c_size_t)]),
    "qt_param_counts": (_ci, [_P(S._Cfg), _ci] + [_P(_u64)] * 6),
    "qt_memory_breakdown": (_ci, [_P(S._Cfg), _P(S._Prec), _P(S._Plan), _ci, _ci, _P(_Tier), _P(_Tier)]),
    "qt_flop_breakdown": (_ci, [_P(S._Cfg), _ci, _ci, _P(_Flops)]),
    "qt_lower_bound_seconds_per_token": (_ci, [_P(_Flops), _P(S._Prec), _P(HardwareProfile), _ci, _ci,
                                               _P(C.c_double)]),
    "qt_mfu": (_ci, [C.c_double, _P(S._Cfg), _P(S._Prec), _P(HardwareProfile), _ci, _P(C.c_double)]),
    "qt_fp8_speedup_ceiling": (_ci, [_P(S._Cfg), _P(HardwareProfile), _ci, _P(C.c_double)]),
    "qt_estimate_step_time": (_ci, [_P(S._Cfg), _P(S._Prec), _P(S._Plan), _P(HardwareProfile), _ci, _ci,
                                    _P(_Time)]),
    "qt_search_plan": (_ci, [_P(S._Cfg), _P(HardwareProfile), _ci, _i64, _ci, _ci, _ci, _ci, _vp, C.c_size_t,
                             _P(C.c_size_t)]),
    "qt_plan_residency": (_ci, [_P(S._Cfg), _P(S._Prec), _P(S._Plan), _u64, _ci, _vp, C.c_size_t,
                                _P(C.c_size_t)]),
    "qt_transfer_time": (_ci, [_u64, _P(HardwareProfile), _ci, _P(C.c_double)]),
    "qt_session_footprint": (_ci, [_P(S._Cfg), _P(S._Prec), _P(S._Plan), _ci, _P(_u64), _P(_u64)]),
    "qt_search_plan_session": (_ci, [_P(S._Cfg), _P(HardwareProfile), _ci, _i64, _ci, _ci, _vp, C.c_size_t,
                                     _P(C.c_size_t)]),
}
_bound = None


def _lib():
    global _bound
    if _bound is None:
        from . import _lib as L
        l = L.lib()
        for n, (rt, at) in _SIGS.items():
            f = getattr(l, n)
            f.restype = rt
            f.argtypes = at
        _bound = l
    return _bound


class PlanError(ValueError):
    pass


def _chk(rc: int) -> None:
    if rc == 1:
        raise PlanError(_lib().qt_plan_last_error().decode())
    if rc != 0:
        raise RuntimeError(_lib().qt_plan_last_error().decode())


def _text(fn, *args) -> str:
    need = C.c_size_t(0)
    _chk(fn(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _chk(fn(*args, buf, need.value, C.byref(need)))
    return buf.value.decode()


# ------------------------------------------------------------------ profiles
def profile_by_name(name: str) -> HardwareProfile:
    p = HardwareProfile()
    _chk(_lib().qt_profile_by_name(name.encode(), C.byref(p)))
    return p


def load_profile(name_or_path: str) -> HardwareProfile:
    p = HardwareProfile()
    _chk(_lib().qt_profile_load(name_or_path.encode(), C.byref(p)))
    return p


def profile_to_json(p: HardwareProfile) -> str:
    return _text(_lib().qt_profile_to_json, C.byref(p))


def profile_from_json(text: str) -> HardwareProfile:
    p = HardwareProfile()
    _chk(_lib().qt_profile_from_json(text.encode(), C.byref(p)))
    return p


# ------------------------------------------------------------------ plan structs
def _cfg(cfg: S.ModelConfig):
    return S._Cfg(*cfg.as_list())


def _prec(block_matmuls="fp8", backward_grads="e4m3", f32_debug=False):
    return S._Prec(0 if block_matmuls == "fp8" else 1, 0 if backward_grads == "e4m3" else 1, int(f32_debug))


def _plan(plan: S.RunPlan):
    return S._Plan(plan.micro_batch, plan.ga_steps, S.recompute_bits(plan.recompute), plan.lmhead_chunk_tokens,
                   plan.attn_chunk_rows, int(plan.shard_weights), int(plan.shard_grads),
                   int(plan.moments == "bf16_sr"), S.offload_bits(plan.offload),
                   0 if plan.transfer_policy == "zero_copy" else 1)


@dataclass
class MemoryBreakdown:
    device: dict
    host: dict


def param_counts(cfg: S.ModelConfig, tied: bool = False) -> dict:
    vals = [_u64() for _ in range(6)]
    _chk(_lib().qt_param_counts(C.byref(_cfg(cfg)), int(tied), *[C.byref(v) for v in vals]))
    return dict(zip(("total", "block_linear", "per_layer_linear", "lmhead", "embed", "norms"), (v.value for v in vals)))


def memory_breakdown(cfg: S.ModelConfig, plan: S.RunPlan, workers: int = 1, tied: bool = False,
                     block_matmuls: str = "fp8") -> MemoryBreakdown:
    d, h = _Tier(), _Tier()
    _chk(_lib().qt_memory_breakdown(C.byref(_cfg(cfg)), C.byref(_prec(block_matmuls)), C.byref(_plan(plan)),
                                    workers, int(tied), C.byref(d), C.byref(h)))
    return MemoryBreakdown({f: getattr(d, f) for f in TIER_FIELDS}, {f: getattr(h, f) for f in TIER_FIELDS})


def flop_breakdown(cfg: S.ModelConfig, recompute=(), tied: bool = False) -> dict:
    f = _Flops()
    _chk(_lib().qt_flop_breakdown(C.byref(_cfg(cfg)), S.recompute_bits(recompute), int(tied), C.byref(f)))
    return {k: getattr(f, k) for k, _ in _Flops._fields_}


def mfu(measured_tps: float, cfg: S.ModelConfig, hw: HardwareProfile, block_matmuls: str = "fp8",
        tied: bool = False) -> float:
    out = C.c_double()
    _chk(_lib().qt_mfu(measured_tps, C.byref(_cfg(cfg)), C.byref(_prec(block_matmuls)), C.byref(hw), int(tied),
                       C.byref(out)))
    return out.value


def fp8_speedup_ceiling(cfg: S.ModelConfig, hw: HardwareProfile, tied: bool = False) -> float:
    out = C.c_double()
    _chk(_lib().qt_fp8_speedup_ceiling(C.byref(_cfg(cfg)), C.byref(hw), int(tied), C.byref(out)))
    return out.value


def estimate_step_time(cfg: S.ModelConfig, plan: S.RunPlan, hw: HardwareProfile, workers: int = 1,
                       tied: bool = False, block_matmuls: str = "fp8") -> dict:
    t = _Time()
    _chk(_lib().qt_estimate_step_time(C.byref(_cfg(cfg)), C.byref(_prec(block_matmuls)), C.byref(_plan(plan)),
                                      C.byref(hw), workers, int(tied), C.byref(t)))
    return {k: getattr(t, k) for k, _ in _Time._fields_}


def search_plan(cfg: S.ModelConfig, hw: HardwareProfile, workers: int, target_batch_tokens: int,
                block_matmuls: str = "fp8", exhaustive: bool = False, tied: bool = False,
                max_results: int = 0) -> dict:
    return json.loads(_text(_lib().qt_search_plan, C.byref(_cfg(cfg)), C.byref(hw), workers, target_batch_tokens,
                            0 if block_matmuls == "fp8" else 1, int(exhaustive), int(tied), max_results))


def plan_residency(cfg: S.ModelConfig, plan: S.RunPlan, device_budget: int, tied: bool = False,
                   block_matmuls: str = "fp8") -> dict:
    return json.loads(_text(_lib().qt_plan_residency, C.byref(_cfg(cfg)), C.byref(_prec(block_matmuls)),
                            C.byref(_plan(plan)), device_budget, int(tied)))


def transfer_time(nbytes: int, hw: HardwareProfile, policy: str = "double_buffer") -> float:
    out = C.c_double()
    _chk(_lib().qt_transfer_time(nbytes, C.byref(hw), 0 if policy == "zero_copy" else 1, C.byref(out)))
    return out.value


def session_footprint(cfg: S.ModelConfig, plan: S.RunPlan, world: int = 1,
                      backward_grads: str = "e5m2") -> tuple[int, int]:
    """Exact (device, pinned host) bytes qt_session_create allocates for this shape."""
    d, h = _u64(), _u64()
    _chk(_lib().qt_session_footprint(C.byref(_cfg(cfg)), C.byref(_prec("fp8", backward_grads)), C.byref(_plan(plan)),
                                     world, C.byref(d), C.byref(h)))
    return d.value, h.value


def search_plan_session(cfg: S.ModelConfig, hw: HardwareProfile, workers: int, target_batch_tokens: int,
                        exhaustive: bool = False, max_results: int = 0) -> dict:
    return json.loads(_text(_lib().qt_search_plan_session, C.byref(_cfg(cfg)), C.byref(hw), workers,
                            target_batch_tokens, int(exhaustive), max_results))
