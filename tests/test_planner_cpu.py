"""Planner parity (CPU): the product planner (csrc/planner.cpp through
paper_2512_15306_b200/planner.py) against the unmodified reference
(oracle/_ref: src/memplan.cpp, src/profiles.cpp, src/offload.cpp) on the same
inputs — byte counts and residency schedules equal, FLOPs / times / MFU equal
to the last bit (same double arithmetic), search rankings identical — plus the
B200 profile and the session-footprint search.

Reference tests mirrored: tests/test_memplan.cpp is absent from the reference
tree, so the cases are the survey's configs (§8d) plus the
reference presets (src/memplan.cpp:98-108)."""
import itertools
import json

import pytest

from paper_2512_15306_b200 import planner as PL
from paper_2512_15306_b200 import session as S

PRESETS = {  # (n_layers, d_model, d_ff, n_heads, n_kv_heads, vocab, seq_len) of src/memplan.cpp:98-108
    "toy": (2, 64, 256, 4, 2, 512, 128),
    "0.5b": (24, 896, 9728, 14, 2, 151936, 1024),
    "1.5b": (28, 1536, 17920, 12, 2, 151936, 1024),
    "7b": (28, 3584, 37888, 28, 4, 152064, 1024),
    "14b": (48, 5120, 27648, 40, 8, 152064, 1024),
    "llama7b": (32, 4096, 22016, 32, 32, 32000, 1024),
}
REF_PROFILES = ("rtx5060ti", "rtx4090", "l40s", "h100", "dgx_spark")


def _cfg(c7):
    return S.ModelConfig(*c7)


def _plan(mb=1, ga=1, rc=0, ob=0, sw=False, sg=False, bf16_moments=True, lm=512, at=256):
    names_rc = [n for i, n in enumerate(S.RECOMPUTE_SITES) if rc >> i & 1]
    names_ob = [n for i, n in enumerate(S.OFFLOAD_CATS) if ob >> i & 1]
    return S.RunPlan(micro_batch=mb, ga_steps=ga, recompute=tuple(names_rc), offload=tuple(names_ob),
                     shard_weights=sw, shard_grads=sg, moments="bf16_sr" if bf16_moments else "f32",
                     lmhead_chunk_tokens=lm, attn_chunk_rows=at)


PLANS = [dict(mb=mb, ga=ga, rc=rc, ob=ob, sw=sw, sg=sg, bf16_moments=bm, lm=lm, at=at)
         for mb, ga, rc, ob, (sw, sg), bm, (lm, at) in [
             (1, 1, 0, 0, (False, False), True, (512, 256)),
             (16, 1, 0, 0, (False, False), False, (0, 0)),
             (8, 4, 1 << 5, 0, (True, True), True, (512, 256)),
             (4, 2, 0b11001, 0b110, (True, False), False, (256, 128)),
             (2, 8, 0b00110, 0b111111, (False, True), True, (100000, 5000)),
             (3, 1, 0b1, 0b011011, (True, True), False, (512, 256)),
         ]]


def _ref_plan(p):
    return dict(mb=p["mb"], ga=p["ga"], recompute_bits=p["rc"], offload_bits=p["ob"], shard_weights=p["sw"],
                shard_grads=p["sg"], bf16_moments=p["bf16_moments"], lmhead_chunk=p["lm"], attn_chunk=p["at"])


@pytest.mark.parametrize("preset", sorted(PRESETS))
@pytest.mark.parametrize("workers", [1, 2, 8])
@pytest.mark.parametrize("tied", [False, True])
def test_memory_breakdown_matches_reference(ref, preset, workers, tied):
    c7 = PRESETS[preset]
    for p in PLANS:
        for bf16 in (False, True):
            got = PL.memory_breakdown(_cfg(c7), _plan(**p), workers, tied, "bf16" if bf16 else "fp8")
            dev, host = ref.memory_breakdown(c7, workers, tied, bf16=bf16, **_ref_plan(p))
            assert got.device == dev, (preset, p, bf16)
            assert got.host == host, (preset, p, bf16)


@pytest.mark.parametrize("preset", sorted(PRESETS))
def test_flops_mfu_ceiling_match_reference(ref, preset):
    c7 = PRESETS[preset]
    cfg = _cfg(c7)
    for rc, tied in itertools.product([0, 1, 0b110, 0b11000, 1 << 5, 0b11111], [False, True]):
        names = [n for i, n in enumerate(S.RECOMPUTE_SITES) if rc >> i & 1]
        assert PL.flop_breakdown(cfg, names, tied) == ref.flop_breakdown(c7, rc, tied)
    for prof in REF_PROFILES:
        hw = PL.profile_by_name(prof)
        for tps in (1.0, 4300.0, 47000.0):
            for bf16 in (False, True):
                assert PL.mfu(tps, cfg, hw, "bf16" if bf16 else "fp8") == ref.mfu(tps, c7, prof, bf16)
        assert PL.fp8_speedup_ceiling(cfg, hw) == ref.fp8_speedup_ceiling(c7, prof)


def test_paper_mfu_anchors(ref):
    """mfu(4300, "7b", FP8, rtx4090) = 0.611 and mfu(47000, "0.5b") = 0.575."""
    hw = PL.profile_by_name("rtx4090")
    assert abs(PL.mfu(4300, _cfg(PRESETS["7b"]), hw) - 0.611) < 1e-3
    assert abs(PL.mfu(47000, _cfg(PRESETS["0.5b"]), hw, tied=True) - 0.575) < 1e-3


@pytest.mark.parametrize("preset", ["toy", "0.5b", "7b", "14b", "llama7b"])
@pytest.mark.parametrize("workers", [1, 4])
def test_estimate_step_time_matches_reference(ref, preset, workers):
    c7 = PRESETS[preset]
    for prof in REF_PROFILES:
        hw = PL.profile_by_name(prof)
        for p in PLANS:
            got = PL.estimate_step_time(_cfg(c7), _plan(**p), hw, workers)
            want = ref.estimate_step_time(c7, prof, workers, **_ref_plan(p))
            got["feasible_in_time"] = float(got["feasible_in_time"])
            assert got == want, (prof, p)


@pytest.mark.parametrize("preset,prof,workers,target", [
    ("toy", "rtx4090", 1, 4096), ("0.5b", "rtx4090", 1, 65536), ("1.5b", "rtx5060ti", 1, 32768),
    ("7b", "rtx4090", 4, 131072), ("14b", "h100", 8, 1 << 20), ("7b", "dgx_spark", 1, 8192)])
def test_search_plan_matches_reference(ref, preset, prof, workers, target):
    c7 = PRESETS[preset]
    tied = preset in ("0.5b", "1.5b")
    got = PL.search_plan(_cfg(c7), PL.profile_by_name(prof), workers, target, tied=tied)
    want = ref.search_plan(c7, prof, workers, target, tied=tied)
    assert [f["plan"]["str"] for f in got["feasible"]] == [f["str"] for f in want["feasible"]]
    assert [f["time"]["tokens_per_second"] for f in got["feasible"]] == [f["tps"] for f in want["feasible"]]
    assert [f["device"]["total"] for f in got["feasible"]] == [f["device"] for f in want["feasible"]]
    assert got.get("no_fit_reason") == want.get("no_fit_reason")


def test_search_plan_exhaustive_and_no_fit(ref):
    c7 = PRESETS["toy"]
    got = PL.search_plan(_cfg(c7), PL.profile_by_name("rtx5060ti"), 2, 8192, exhaustive=True)
    want = ref.search_plan(c7, "rtx5060ti", 2, 8192, exhaustive=True)
    assert [f["plan"]["str"] for f in got["feasible"]] == [f["str"] for f in want["feasible"]]
    big = (64, 8192, 65536, 64, 8, 152064, 1024)
    got = PL.search_plan(_cfg(big), PL.profile_by_name("rtx5060ti"), 1, 8192)
    want = ref.search_plan(big, "rtx5060ti", 1, 8192)
    assert got["feasible"] == [] and want["feasible"] == []
    assert got["no_fit_reason"] == want["no_fit_reason"]


def _events_jsonl(events):
    # to_jsonl (src/offload.cpp:145-160) field order: time, kind, category, layer, buffer, bytes, resident
    out = []
    for e in events:
        t = e["time"]
        ts = str(int(t)) if float(t).is_integer() else repr(t)
        out.append('{"time":%s,"kind":"%s","category":"%s","layer":%d,"buffer":%d,"bytes":%d,"resident":%d}'
                   % (ts, e["kind"], e["category"], e["layer"], e["buffer"], e["bytes"], e["resident"]))
    return "".join(x + "\n" for x in out)


@pytest.mark.parametrize("preset", ["toy", "0.5b", "7b"])
def test_plan_residency_matches_reference(ref, preset):
    c7 = PRESETS[preset]
    for p in PLANS:
        for budget in (16 << 30, 80 << 30):
            got = PL.plan_residency(_cfg(c7), _plan(**p), budget)
            want = ref.plan_residency(c7, budget, **_ref_plan(p))
            assert _events_jsonl(got["events"]) == want["jsonl"], p
            assert got["high_water_device"] == want["high_water"]
            assert got["high_water_weights"] == want["hw_weights"]
            assert got["high_water_grads"] == want["hw_grads"]
            assert got["high_water_residuals"] == want["hw_residuals"]
            assert got["feasible"] == want["feasible"]
            assert got.get("report", "") == want["report"]


def test_profiles_match_reference_and_roundtrip(ref):
    for prof in REF_PROFILES:
        p = PL.profile_by_name(prof)
        assert json.loads(PL.profile_to_json(p)) == ref.profile_json(prof)
        q = PL.profile_from_json(PL.profile_to_json(p))
        assert bytes(q) == bytes(p)
        for nbytes in (0, 1 << 20, 7 << 30):
            for zc in (True, False):
                assert PL.transfer_time(nbytes, p, "zero_copy" if zc else "double_buffer") == \
                    ref.transfer_time(nbytes, prof, zc)
    with pytest.raises(PL.PlanError, match="unknown hardware profile 'nope'; available: rtx5060ti"):
        PL.profile_by_name("nope")


def test_b200_profile_and_mfu():
    hw = PL.profile_by_name("b200")
    assert hw.device_bytes == 180_000_000_000 and hw.p2p == 1
    assert hw.peak_flops_fp8 == 4.5e15 and hw.peak_flops_bf16 == 2.25e15
    # 40 % MFU at the Llama-7B shape = 42.8k tokens/s
    m = PL.mfu(42_800, _cfg(PRESETS["llama7b"]), hw)
    assert 0.39 < m < 0.41, m


def test_session_footprint_and_session_search():
    """The B200 search filters by the session's own arena (exact bytes of
    qt_session_create), which is larger than the reference's estimate (the
    session keeps f32 logits and the unrounded attention output)."""
    cfg = _cfg(PRESETS["0.5b"])
    dev, host = PL.session_footprint(cfg, _plan(mb=16, bf16_moments=False, lm=0, at=0))
    est = PL.memory_breakdown(cfg, _plan(mb=16, bf16_moments=False, lm=0, at=0), tied=False)
    assert 40e9 < dev < 60e9, dev
    assert dev > sum(est.device.values()) * 0.5
    hw = PL.profile_by_name("b200")
    res = PL.search_plan_session(_cfg(PRESETS["llama7b"]), hw, 1, 8 * 1024, max_results=5)
    assert res["feasible"], res
    for f in res["feasible"]:
        assert f["device_bytes"] <= hw.device_bytes


def test_session_footprint_sharding_switches_save_memory():
    """Qwen2.5-14B shape at W = 8 (BASELINE config 5): shard_weights keeps 1/8 of the bf16
    block weights and streams the FP8 codes per layer; shard_grads reduce-scatters per layer
    instead of holding the full gradient and receive buffers; offload.weights moves the
    codes to pinned host memory.  Each switch lowers the session's real device arena."""
    cfg = _cfg(PRESETS["14b"])
    base = dict(mb=4, bf16_moments=True, lm=0, at=0)

    def fp(**kw):
        return PL.session_footprint(cfg, _plan(**{**base, **kw}), world=8)

    d0, _ = fp()
    d_sw, _ = fp(sw=True)
    d_sg, _ = fp(sg=True)
    d_both, _ = fp(sw=True, sg=True)
    d_off, h_off = fp(sw=True, sg=True, ob=1 << 4)
    gb = 1e9
    assert d0 - d_sw > 30 * gb, (d0, d_sw)      # bf16 slices (23 GB) + codes (11 GB)
    assert d0 - d_sg > 45 * gb, (d0, d_sg)      # gradients (25 GB) + receive buffer (25 GB)
    assert d0 - d_both > 80 * gb, (d0, d_both)
    assert d_off <= d_both and h_off > 13 * gb  # the host weight cache holds every layer's codes
    assert d_both < 0.5 * d0, (d0 / gb, d_both / gb)
