"""The multi-rank product code executed on ONE GPU: W sessions of an in-process
worker group (qt_group_create; the reference's WorkerGroup, src/comms.cpp:19-38),
one host thread each, whose collectives are copy-engine pulls between their
arenas (csrc/transport.cuh PeerTransport).  This runs the session's own
ZeRO-1 code — the bf16 shard all-to-all + ascending-rank f32 sum
(reduce_tensors / ordered_sum_kernel), the norm all-reduce, AdamW on the rank's
256*W-aligned slice, the in-place all-gathers, the per-layer exchange of
shard_grads and the E4M3-code all-gather of shard_weights — and checks it:

* bitwise, against the reference's ZeRO-1 arithmetic applied on the host to
  the ranks' own local gradient accumulators: ascending-worker f32 sum
  (src/trainer.cpp:90-103), adamw_tensor of the reference on every tensor
  (src/optim.cpp:37-70, 112-176) — updated params and moment slices equal bit
  for bit, on every rank;
* bitwise across the sharding switches (RunPlan::shard_grads / shard_weights
  only change where bytes live, not the arithmetic);
* within the one-step tolerances, against the reference trainer step with
  W workers (ref_model_train_step(..., workers=W), src/trainer.cpp:64-110).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = dict(n_layers=2, d_model=128, d_ff=256, n_heads=2, n_kv_heads=1, vocab=256, seq_len=64)
B = 2


def _tokens(vocab, batch, seq, seed):
    g = np.random.default_rng(seed)
    return g.integers(0, vocab, size=batch * (seq + 1), dtype=np.int32)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _group(W, ga=1, sg=False, sw=False, seed=1234, params=None, offload=()):
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)
    grp = S.WorkerGroup(W)
    plan = S.RunPlan(micro_batch=B, ga_steps=ga, shard_grads=sg, shard_weights=sw, offload=offload)
    ss = [S.Session(cfg, plan=plan, seed=seed, rank=r, group=grp) for r in range(W)]
    for s in ss:
        assert s.transport == "peer-copy"
        for n, v in params.items():
            s.upload(n, v)
    return cfg, grp, ss


def _step_tokens(cfg, W, ga, step):
    """GA x W micro-batches ordered (ga, w) as trainer.cpp:75-76; rank w gets its GA."""
    mbs = [[_tokens(cfg.vocab, B, cfg.seq_len, 1000 * step + 10 * g + w) for w in range(W)] for g in range(ga)]
    flat = np.concatenate([mbs[g][w] for g in range(ga) for w in range(W)])
    per_rank = [np.concatenate([mbs[g][w] for g in range(ga)]) for w in range(W)]
    return flat, per_rank


def _run(grp, ss, per_rank, step, max_norm):
    return grp.run(lambda r, t: ss[r].train_step(t, B, step=step, max_grad_norm=max_norm), per_rank)


# shard_grads keeps no local accumulator for layer tensors (it reduce-scatters them per layer);
# its arithmetic is checked bitwise against these runs in test_sharding_switches_bitwise_invariant
CASES = [(2, 1, False, False), (2, 2, False, False), (3, 1, False, False), (4, 1, False, False),
         (2, 1, False, True), (2, 2, False, True), (4, 1, False, True)]


@pytest.mark.parametrize("W,ga,sg,sw", CASES)
def test_zero1_step_bitwise_vs_reference_arithmetic(ref, W, ga, sg, sw):
    rm = ref.RefModel(list(SMALL.values()), 1234)
    params = {n: rm.get(n) for n in rm.names}
    cfg, grp, ss = _group(W, ga, sg, sw, params=params)
    names = ss[0].names
    state = {n: (params[n], np.zeros_like(params[n]), np.zeros_like(params[n])) for n in names}
    for step in range(2):
        _, per_rank = _step_tokens(cfg, W, ga, step)
        res = _run(grp, ss, per_rank, step, 0.0)  # max_grad_norm 0: no clip (optim.cpp:107-110)
        norms = {r[1] for r in res}
        assert len(norms) == 1, norms  # every rank saw the same all-reduced norm
        acc = {n: [s.grad(n) for s in ss] for n in names}  # each rank's local GradAccumulator
        ssq = 0.0
        for n in sorted(names):  # global_grad_norm: std::map (name) order, 256-element blocks
            g = acc[n][0].copy()
            for w in range(1, W):
                g = (g + acc[n][w]).astype(np.float32)  # ascending-worker f32 sum, trainer.cpp:95-102
            ssq += ref.grad_norm_partials(g)
            p, m, v = ref.adamw_tensor(n, *state[n], g, lr=1e-3, seed=1234, step_count=step,
                                       grad_scale=1.0 / (ga * W))
            state[n] = (p, m, v)
        assert abs(np.sqrt(ssq) / (ga * W) - next(iter(norms))) <= 1e-6 * np.sqrt(ssq) / (ga * W)
        for n in names:
            p, m, v = state[n]
            for r, s in enumerate(ss):
                np.testing.assert_array_equal(s.download(n), p, err_msg=f"step {step} rank {r} {n}")
            # moment slices: rank w owns [w*pw, (w+1)*pw) (shard_layout, comms.cpp:69-73)
            from paper_2512_15306_b200 import session as S
            _, pw = S.shard_layout(p.size, W)
            for r, s in enumerate(ss):
                gm, gv = s.moments(n)
                lo, hi = min(r * pw, p.size), min((r + 1) * pw, p.size)
                np.testing.assert_array_equal(gm, m[lo:hi], err_msg=f"m rank {r} {n}")
                np.testing.assert_array_equal(gv, v[lo:hi], err_msg=f"v rank {r} {n}")


SWITCHES = [(False, False, ()), (True, False, ()), (False, True, ()), (True, True, ()),
            (False, False, ("weights",)), (False, True, ("weights",)), (True, True, ("weights",))]


@pytest.mark.parametrize("W,ga", [(2, 1), (2, 2), (4, 1)])
def test_sharding_switches_bitwise_invariant(ref, W, ga):
    """RunPlan::shard_grads (per-layer reduce-scatter into the rank's shard, no full local
    gradient buffer), shard_weights (the rank keeps its slice of the bf16 block weights; the
    FP8 codes are all-gathered one layer ahead) and offload.weights (codes in pinned host
    memory, two device layer slots; with shard_weights the host weight cache) change where
    bytes live, not the arithmetic: params, moments and losses bitwise equal to plain ZeRO-1.
    Exception: shard_grads with GA > 1 reduces every micro-batch, so the
    summation order differs; those runs meet the one-step rules instead."""
    rm = ref.RefModel(list(SMALL.values()), 77)
    params = {n: rm.get(n) for n in rm.names}
    outs = []
    for sg, sw, off in SWITCHES:
        cfg, grp, ss = _group(W, ga, sg, sw, seed=77, params=params, offload=off)
        losses = []
        for step in range(3):
            _, per_rank = _step_tokens(cfg, W, ga, step)
            losses.append(_run(grp, ss, per_rank, step, 1.0))
        red = {n: ss[0].reduced_grad(n) for n in ss[0].names}
        mom = {n: [s.moments(n) for s in ss] for n in ss[0].names}
        outs.append((sg, losses, {n: ss[0].download(n) for n in ss[0].names}, red, mom))
        for s in ss:
            s.close()
    base = outs[0]
    for (sg, losses, p, red, mom), sw_ in zip(outs[1:], SWITCHES[1:]):
        if sg and ga > 1:
            for st0, st1 in zip(base[1], losses):
                (l0, n0), (l1, n1) = st0[0], st1[0]
                assert abs(l0 - l1) <= 1e-3 * abs(l0) and abs(n0 - n1) <= 2e-2 * n0, (sw_, st0, st1)
            for n in p:
                assert _rel(p[n], base[2][n]) < 4e-3, (sw_, n)
            continue
        assert losses == base[1], sw_
        for n in p:
            np.testing.assert_array_equal(p[n], base[2][n], err_msg=f"{sw_} {n}")
            np.testing.assert_array_equal(red[n], base[3][n], err_msg=f"{sw_} reduced grad {n}")
            for (m0, v0), (m1, v1) in zip(base[4][n], mom[n]):
                np.testing.assert_array_equal(m1, m0, err_msg=f"{sw_} m {n}")
                np.testing.assert_array_equal(v1, v0, err_msg=f"{sw_} v {n}")


def test_offload_weights_single_gpu_bitwise():
    """offload.weights on one rank (codes in pinned host memory, streamed per layer into two
    device slots) is bitwise the resident-codes step, and frees the codes' device bytes."""
    from paper_2512_15306_b200 import planner as PL
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)
    res = []
    for off in ((), ("weights",)):
        s = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), S.RunPlan(micro_batch=B, offload=off), seed=9)
        s.init_params(9)
        losses = [s.train_step(_tokens(cfg.vocab, B, cfg.seq_len, 50 + k), B, step=k) for k in range(3)]
        res.append((losses, {n: s.download(n) for n in s.names}, [s.weight_codes(l, k) for l in range(2)
                                                                   for k in range(4)]))
        s.close()
    assert res[0][0] == res[1][0]
    for n in res[0][1]:
        np.testing.assert_array_equal(res[0][1][n], res[1][1][n], err_msg=n)
    for a, b in zip(res[0][2], res[1][2]):
        np.testing.assert_array_equal(a, b)
    big = S.ModelConfig(n_layers=48, d_model=5120, d_ff=27648, n_heads=40, n_kv_heads=8, vocab=152064, seq_len=1024)
    d0, _ = PL.session_footprint(big, S.RunPlan(micro_batch=1, moments="bf16_sr"))
    d1, h1 = PL.session_footprint(big, S.RunPlan(micro_batch=1, moments="bf16_sr", offload=("weights",)))
    assert d0 - d1 > 12e9 and h1 > 12e9, (d0, d1, h1)  # 13.2 GB of E4M3 codes move to the host


@pytest.mark.parametrize("W,ga", [(2, 1), (4, 2)])
def test_group_step_vs_reference_trainer(ref, W, ga):
    """One-step rules against the reference trainer with W
    workers: loss 1e-3, norm 2e-2, updated params <= 4e-3 norm-wise."""
    rm = ref.RefModel(list(SMALL.values()), 1234)
    params = {n: rm.get(n) for n in rm.names}
    cfg, grp, ss = _group(W, ga, sg=True, sw=True, params=params)
    flat, per_rank = _step_tokens(cfg, W, ga, 0)
    lw, nw = rm.train_step(flat, B, ga_steps=ga, workers=W, step=0)
    res = _run(grp, ss, per_rank, 0, 1.0)
    lg = float(np.mean([r[0] for r in res]))
    ng = res[0][1]
    assert abs(lg - lw) / lw < 1e-3, (lg, lw)
    assert abs(ng - nw) / nw < 2e-2, (ng, nw)
    for n in rm.names:
        r = _rel(ss[0].download(n), rm.get(n))
        assert r < 4e-3, (n, r)
