"""Offload tiers on the device path (RunPlan::offload, include/qtrain/memplan.hpp:
34-52): optimizer moments (m, v), the bf16 master block
weights, the gradient buffer, the residual stream (x) and the FP8 weight codes
placed in pinned host memory, with the zero-copy and the double-buffer
transfer policies.  The reference only simulates residency (src/offload.cpp);
here the bytes really move, so the check is that they move without changing
the arithmetic: losses, norms, updated params, moments and weight codes are
bit-for-bit those of the all-resident session, on one rank and on a 2-rank
peer group with ZeRO-1 sharding."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = dict(n_layers=3, d_model=128, d_ff=256, n_heads=2, n_kv_heads=1, vocab=256, seq_len=64)
B = 2


def _tokens(vocab, batch, seq, seed):
    return np.random.default_rng(seed).integers(0, vocab, size=batch * (seq + 1), dtype=np.int32)


def _run(offload=(), policy="double_buffer", moments="f32", ga=1, recompute=(), steps=3):
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)
    plan = S.RunPlan(micro_batch=B, ga_steps=ga, moments=moments, offload=offload, transfer_policy=policy,
                     recompute=recompute)
    s = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), plan, seed=21)
    s.init_params(21)
    out = []
    for k in range(steps):
        toks = np.concatenate([_tokens(cfg.vocab, B, cfg.seq_len, 100 * k + g) for g in range(ga)])
        out.append(s.train_step(toks, B, step=k))
    state = {n: (s.download(n), *s.moments(n)) for n in s.names}
    codes = [s.weight_codes(l, k) for l in range(cfg.n_layers) for k in range(4)]
    nbytes = s.device_bytes
    s.close()
    return out, state, codes, nbytes


def _same(a, b, what):
    assert a[0] == b[0], (what, a[0], b[0])
    for n in a[1]:
        for x, y, nm in zip(a[1][n], b[1][n], ("param", "m", "v")):
            np.testing.assert_array_equal(x, y, err_msg=f"{what}: {nm} {n}")
    for x, y in zip(a[2], b[2]):
        np.testing.assert_array_equal(x, y, err_msg=f"{what}: codes")


@pytest.mark.parametrize("moments", ["f32", "bf16_sr"])
@pytest.mark.parametrize("policy", ["zero_copy", "double_buffer"])
def test_offload_tiers_bitwise_one_rank(policy, moments):
    base = _run(moments=moments)
    for off in (("m",), ("v",), ("m", "v"), ("master",), ("grads",), ("x",), ("weights",),
                ("x", "m", "v", "master", "weights", "grads")):
        got = _run(off, policy, moments)
        _same(got, base, f"{off} {policy} {moments}")
        assert got[3] < base[3], (off, got[3], base[3])  # the device arena shrinks


def test_offload_with_recompute_and_accumulation():
    base = _run(ga=2, recompute=("ffn",))
    got = _run(("x", "m", "v", "master", "weights"), "double_buffer", ga=2, recompute=("ffn",))
    _same(got, base, "ga2 + ffn recompute")


@pytest.mark.parametrize("policy", ["zero_copy", "double_buffer"])
def test_offload_tiers_bitwise_two_ranks(policy):
    """2-rank peer group with shard_weights + shard_grads: offloading every tier keeps the
    ZeRO-1 step bitwise (the peer transport reads the ranks' host regions too)."""
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)

    def run(off):
        grp = S.WorkerGroup(2)
        plan = S.RunPlan(micro_batch=B, shard_weights=True, shard_grads=True, offload=off, transfer_policy=policy)
        ss = [S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), plan, seed=3, rank=r, group=grp) for r in range(2)]
        for s in ss:
            s.init_params(3)
        res = []
        for k in range(3):
            toks = [_tokens(cfg.vocab, B, cfg.seq_len, 10 * k + r) for r in range(2)]
            res.append(grp.run(lambda r, t: ss[r].train_step(t, B, step=k), toks))
        params = {n: ss[0].download(n) for n in ss[0].names}
        moms = {n: [s.moments(n) for s in ss] for n in ss[0].names}
        for s in ss:
            s.close()
        return res, params, moms

    a = run(())
    b = run(("x", "m", "v", "master", "weights"))
    assert a[0] == b[0]
    for n in a[1]:
        np.testing.assert_array_equal(a[1][n], b[1][n], err_msg=n)
        for (m0, v0), (m1, v1) in zip(a[2][n], b[2][n]):
            np.testing.assert_array_equal(m0, m1, err_msg=n)
            np.testing.assert_array_equal(v0, v1, err_msg=n)
