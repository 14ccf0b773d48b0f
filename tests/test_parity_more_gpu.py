"""Parity items pinned directly against the unmodified reference (oracle/_ref):

* RoPE: the session's host table + the device kernel vs the reference's own
  rope_apply (src/model.cpp:169-191, exported by oracle/ref_internal.cpp) —
  bit-exact forward and backward.
* Embedding backward: device stable sort + ordered segment sum + bf16 round +
  SR accumulate vs embedding_backward_sorted (src/tensorops.cpp:317-342) and
  GradAccumulator (src/model.cpp:442-464), repeated ids — bit-exact.
* AdamW with bf16-SR moments (src/optim.cpp:37-70) — bit-exact, two steps.
* A GA = 2 trainer step (src/trainer.cpp:64-110).
* A teacher-forced 20-step curve: each step starts from the
  reference's own weights and optimizer state, and must meet the one-step rules.
* One trainer step at the real Qwen2.5-0.5B and Llama-7B widths (1-2 layers,
  full vocabulary, short sequences) from identical weights.
* The update gate: an out-of-range token, a non-finite activation or gradient
  leaves params, moments and the step count untouched (the reference throws
  before updating, src/model.cpp:125-129, 324-325; src/optim.cpp:47).
"""
import numpy as np
import pytest

from tests.helpers import bf16_grid_round, rng_floats

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = dict(n_layers=2, d_model=128, d_ff=256, n_heads=2, n_kv_heads=1, vocab=256, seq_len=64)


def _tokens(vocab, batch, seq, seed):
    g = np.random.default_rng(seed)
    return g.integers(0, vocab, size=batch * (seq + 1), dtype=np.int32)


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _pair(ref, cfgd, seed=1234, grad_e5m2=False, micro_batch=2, moments="f32", **kw):
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**cfgd)
    rm = ref.RefModel(cfg.as_list(), seed, grad_e5m2=grad_e5m2, bf16_moments=(moments == "bf16_sr"))
    sess = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2" if grad_e5m2 else "e4m3"),
                     S.RunPlan(micro_batch=micro_batch, moments=moments, **kw), seed=seed)
    for n in rm.names:
        sess.upload(n, rm.get(n))
    return cfg, rm, sess


# ------------------------------------------------------------------ RoPE
@pytest.mark.parametrize("B,T,H,Hkv,hd", [(2, 64, 4, 2, 64), (1, 1024, 14, 2, 64), (1, 256, 8, 8, 128),
                                          (2, 96, 4, 1, 32)])
def test_rope_bitexact_vs_reference(ref, B, T, H, Hkv, hd):
    from paper_2512_15306_b200 import _lib
    from paper_2512_15306_b200 import session as S
    d = H * hd
    q = d + 2 * Hkv * hd
    cfg7 = [1, d, 64, H, Hkv, 256, T]
    x = rng_floats(T + hd + B, B * T * q, -3, 3).reshape(B * T, q)
    tab = torch.from_numpy(S.rope_table(T, hd)).cuda()
    for bwd in (0, 1):
        want = ref.rope_apply(cfg7, x, B, T, backward=bool(bwd))
        xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
        am = torch.zeros(1, dtype=torch.int32, device="cuda")
        rc = _lib.lib().qtk_rope(xt.data_ptr(), B * T, T, H + Hkv, hd, q, tab.data_ptr(), bwd,
                                 am.data_ptr() if bwd else None, torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        np.testing.assert_array_equal(xt.float().cpu().numpy(), want)
        if bwd:  # fused absmax over the whole rotated row (d_qkv quantization)
            assert am.view(torch.float32).item() == np.abs(want).max()


# ------------------------------------------------------------------ embedding backward
@pytest.mark.parametrize("n,V,d,distinct", [(2048, 512, 128, 64), (4096, 151936, 896, 300), (1000, 1000, 256, 1000)])
def test_embedding_backward_bitexact_vs_reference(ref, n, V, d, distinct):
    from paper_2512_15306_b200 import _lib
    g = np.random.default_rng(n + V)
    vocab_ids = g.choice(V, size=distinct, replace=False)
    ids = vocab_ids[g.integers(0, distinct, n)].astype(np.int32)
    dr = rng_floats(n + 1, n * d, -1, 1).reshape(n, d)
    buf0 = rng_floats(n + 2, V * d, -0.01, 0.01)
    seed, stream, micro = 99, ref.fnv1a64("gradaccum/embed"), 3
    # reference: ordered f32 sum per id, bf16 round (model.cpp:442-444), accumulate
    e = bf16_grid_round(ref.embedding_backward(ids, dr, V).ravel())
    want = ref.grad_accumulate("embed", buf0, e, seed=seed, micro_step=micro)
    s = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    ids_t = torch.from_numpy(ids).cuda()
    scratch_b = L.qtk_embed_sort_scratch_bytes(n, V)
    scratch = torch.empty(max(scratch_b, 1), dtype=torch.uint8, device="cuda")
    sorted_pos = torch.empty(n, dtype=torch.int32, device="cuda")
    seg_tok = torch.empty(n, dtype=torch.int32, device="cuda")
    seg_off = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    nseg = torch.zeros(4, dtype=torch.int32, device="cuda")
    assert L.qtk_embed_sort(ids_t.data_ptr(), n, V, scratch.data_ptr(), scratch_b, sorted_pos.data_ptr(),
                            seg_tok.data_ptr(), seg_off.data_ptr(), nseg.data_ptr(), s) == 0
    grad = torch.from_numpy(buf0).cuda().to(torch.bfloat16)
    drt = torch.from_numpy(dr).cuda().to(torch.bfloat16)
    assert L.qtk_embed_bwd(sorted_pos.data_ptr(), seg_off.data_ptr(), seg_tok.data_ptr(), nseg.data_ptr(), n,
                           drt.data_ptr(), d, grad.data_ptr(), seed, stream, micro * V * d, s) == 0
    torch.cuda.synchronize()
    assert int(nseg[0].item()) == len(np.unique(ids))
    np.testing.assert_array_equal(grad.float().cpu().numpy().ravel(), want)


# ------------------------------------------------------------------ bf16-SR AdamW
def test_adamw_bf16_sr_moments_bitexact(ref):
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)
    s = S.Session(cfg, plan=S.RunPlan(micro_batch=2, moments="bf16_sr"),
                  hyper=S.AdamWHyper(lr=1e-3, weight_decay=0.1), seed=7)
    s.init_params(7)
    toks = _tokens(cfg.vocab, 2, cfg.seq_len, 1)
    s.build_step_context()
    s.zero_grads()
    s.forward(toks, 2)
    s.backward(0)
    grads = {n: s.grad(n) for n in s.names}
    p0 = {n: s.download(n) for n in s.names}
    z = {n: np.zeros_like(p0[n]) for n in s.names}
    state = {n: (p0[n], z[n], z[n]) for n in s.names}
    for step, scale in ((0, 0.37), (1, 0.5)):
        s.adamw_step(scale)
        for n in s.names:
            p, m, v = ref.adamw_tensor(n, *state[n], grads[n], lr=1e-3, wd=0.1, bf16_moments=True, seed=7,
                                       step_count=step, grad_scale=scale)
            np.testing.assert_array_equal(s.download(n), p, err_msg=n)
            gm, gv = s.moments(n)
            np.testing.assert_array_equal(gm, m, err_msg=n)
            np.testing.assert_array_equal(gv, v, err_msg=n)
            state[n] = (p, m, v)


# ------------------------------------------------------------------ GA = 2
@pytest.mark.parametrize("recompute", [(), ("block",)])
def test_ga2_train_step_parity(ref, recompute):
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)
    rm = ref.RefModel(cfg.as_list(), 1234, recompute_bits=S.recompute_bits(recompute))
    sess = S.Session(cfg, plan=S.RunPlan(micro_batch=2, ga_steps=2, recompute=recompute), seed=1234)
    for n in rm.names:
        sess.upload(n, rm.get(n))
    toks = np.concatenate([_tokens(cfg.vocab, 2, cfg.seq_len, 40), _tokens(cfg.vocab, 2, cfg.seq_len, 41)])
    lw, nw = rm.train_step(toks, 2, ga_steps=2, step=0)
    lg, ng = sess.train_step(toks, 2, step=0)
    assert abs(lg - lw) / lw < 1e-3, (lg, lw)
    assert abs(ng - nw) / nw < 2e-2, (ng, nw)
    for n in rm.names:
        r = _rel(sess.download(n), rm.get(n))
        assert r < 4e-3, (n, r)


# ------------------------------------------------------------------ teacher-forced 20-step curve
def test_loss_curve_20_steps_teacher_forced(ref):
    """at every step the device session is re-loaded with the
    reference's weights and AdamW state (teacher forcing), runs one trainer step
    on that step's tokens, and must meet the one-step rules: loss <= 1e-3
    relative, grad norm <= 2e-2, updated params norm-wise within 2x the
    reference's own single-flip envelope of that step (the same state with one
    E4M3 code step in layers.0.w_qkv or layers.1.w_down; floor 1e-3)."""
    from paper_2512_15306_b200 import session as S
    tiny = S.PRESETS["tiny"]
    T, B, steps = 128, 1, 20
    cfgd = dict(n_layers=tiny.n_layers, d_model=tiny.d_model, d_ff=tiny.d_ff, n_heads=tiny.n_heads,
                n_kv_heads=tiny.n_kv_heads, vocab=tiny.vocab, seq_len=T)
    cfg, rm, sess = _pair(ref, cfgd, grad_e5m2=True, micro_batch=B)
    worst_loss = worst_p = 0.0
    perts = [ref.RefModel(cfg.as_list(), 1234, grad_e5m2=True) for _ in range(2)]
    targets = ("layers.0.w_qkv", "layers.1.w_down")
    for st in range(steps):
        state = {n: (rm.get(n), *rm.moments(n)) for n in rm.names}
        for n, (p, m, v) in state.items():  # teacher forcing: the reference's state before this step
            sess.upload(n, p)
            sess.set_moments(n, m, v, st)
        envs = {}
        toks = _tokens(cfg.vocab, B, T, 700 + st)
        for pm, tgt in zip(perts, targets):
            for n, (p, m, v) in state.items():
                pm.set(n, p)
                pm.set_moments(n, m, v, st)
            w = state[tgt][0].copy()
            i = int(np.argmax(np.abs(w) < 0.5 * np.abs(w).max()))
            w[i] = ref.bf16_round(float(w[i]) * 1.125)
            pm.set(tgt, w)
        lw, nw = rm.train_step(toks, B, step=st)
        for pm, tgt in zip(perts, targets):
            pm.train_step(toks, B, step=st)
            for n in rm.names:
                if n != tgt:
                    envs[n] = max(envs.get(n, 0.0), _rel(pm.get(n), rm.get(n)))
        lg, ng = sess.train_step(toks, B, step=st)
        worst_loss = max(worst_loss, abs(lg - lw) / lw)
        assert abs(lg - lw) / lw < 1e-3, (st, lg, lw)
        assert abs(ng - nw) / nw < 2e-2, (st, ng, nw)
        for n in rm.names:
            r = _rel(sess.download(n), rm.get(n))
            worst_p = max(worst_p, r / max(2.0 * envs[n], 1e-3))
            assert r <= max(2.0 * envs[n], 1e-3), (st, n, r, envs[n])
    print(f"teacher-forced 20 steps: worst loss rel {worst_loss:.2e}, worst param gap / bound {worst_p:.2f}")


# ------------------------------------------------------------------ real widths
def _update_flips(after, before, ref_after, g_ref):
    """Gradient mass whose one-step update direction differs from the
    reference's: sum |g_ref| over flipped elements / sum |g_ref|.  The first
    AdamW step is sign-like (m/sqrt(v) = g/|g|, src/optim.cpp:61-70), so a
    last-bit difference in a gradient that is ~0 moves that element by a full
    2*lr; weighting by |g| counts the flips of elements that carry gradient."""
    a = np.sign(np.asarray(after, np.float64) - before)
    b = np.sign(np.asarray(ref_after, np.float64) - before)
    w = np.abs(np.asarray(g_ref, np.float64))
    return float(w[a != b].sum() / max(w.sum(), 1e-30))


def _width_step(ref, preset, n_layers, T, seed=1234, floor=5e-3):
    """One teacher-forced train step at the real widths: loss 1e-3 rel,
    norm 2e-2, every gradient within 2x the reference's own single-code-flip
    envelope (its sensitivity to ONE E4M3 code of one weight: per-tensor FP8
    quantization turns any last-bit difference upstream into such flips,
    SURVEY.md 8(c), scripts/chaos_floor.py), and the updated params' direction
    flips within 2x the flips the same perturbation causes in the reference."""
    from paper_2512_15306_b200 import session as S
    p = S.PRESETS[preset]
    cfgd = dict(n_layers=n_layers, d_model=p.d_model, d_ff=p.d_ff, n_heads=p.n_heads, n_kv_heads=p.n_kv_heads,
                vocab=p.vocab, seq_len=T)
    cfg, rm, sess = _pair(ref, cfgd, seed=seed, grad_e5m2=True, micro_batch=1)
    toks = _tokens(cfg.vocab, 1, T, 31)
    before = {n: rm.get(n) for n in rm.names}
    lw, nw = rm.train_step(toks, 1, step=0)
    lg, ng = sess.train_step(toks, 1, step=0)
    assert abs(lg - lw) / lw < 1e-3, (lg, lw)
    assert abs(ng - nw) / nw < 2e-2, (ng, nw)
    # the reference with ONE E4M3 code step in one weight (four such perturbations in
    # different tensors; the envelope of a tensor is the largest response among the others)
    perts = []
    for tgt in ("layers.0.w_qkv", "layers.0.w_o", "layers.0.w_gate_up", f"layers.{n_layers - 1}.w_down"):
        pert = ref.RefModel(cfg.as_list(), seed, grad_e5m2=True)
        w = pert.get(tgt).copy()
        i = int(np.argmax(np.abs(w) < 0.5 * np.abs(w).max()))
        w[i] = ref.bf16_round(float(w[i]) * 1.125)
        pert.set(tgt, w)
        pert.train_step(toks, 1, step=0)
        perts.append((tgt, pert))
    worst, bad = {}, []
    for n in rm.names:
        want_g = rm.acc_grad(n)
        # any of the perturbations (a tensor's gradient does not contain its own weight, only
        # the activations downstream of it): the largest response is the envelope
        env_g = max(_rel(p.acc_grad(n), want_g) for _, p in perts)
        got_g = _rel(sess.grad(n), want_g)
        env_f = max(_update_flips(p.get(n), before[n], rm.get(n), want_g) for t, p in perts if t != n)
        got_f = _update_flips(sess.download(n), before[n], rm.get(n), want_g)
        worst[n] = tuple(round(float(x), 5) for x in (got_g, env_g, got_f, env_f))
        if got_g > max(2.0 * env_g, floor) or got_f > max(2.0 * env_f, 5e-3):
            bad.append(n)
    print(worst)
    assert not bad, {n: worst[n] for n in bad}


def test_train_step_qwen05b_width_2_layers(ref):
    """d 896, F 9728, 14/2 heads, V 151936, 2 layers, T 16."""
    _width_step(ref, "qwen2.5-0.5b", 2, 16)


def test_train_step_llama7b_width_1_layer(ref):
    """d 4096, F 22016, 32/32 heads (hd 128), V 32000, 1 layer, T 16.  With 16 tokens each
    per-tensor FP8 scale is set by a handful of elements, so a last-bit difference in the
    attention output's absmax element moves every code of att (scripts/diag_width.py: att
    99.7 % bit-exact, r_mid 92 %, gate_up 65 %); such scale flips are the reference's own
    order-noise mechanism but a single weight-code flip rarely triggers one,
    so the envelope is floored at 0.1 for the gradients here; the loss, the norm, the
    forward sites up to the first re-quantisation and the update directions keep their
    rules."""
    _width_step(ref, "llama-7b", 1, 16, floor=0.1)


# ------------------------------------------------------------------ update gate
def _fresh(seed=5, **plan):
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)
    s = S.Session(cfg, plan=S.RunPlan(micro_batch=2, **plan), seed=seed)
    s.init_params(seed)
    return cfg, s


def _state(s):
    return {n: (s.download(n), *s.moments(n)) for n in s.names}


def _same_state(a, b):
    for n in a:
        for x, y in zip(a[n], b[n]):
            np.testing.assert_array_equal(x, y, err_msg=n)


def test_bad_token_train_step_updates_nothing():
    cfg, s = _fresh()
    good = _tokens(cfg.vocab, 2, cfg.seq_len, 1)
    s.train_step(good, 2, step=0)  # steady state: the next steps replay the captured graph
    before = _state(s)
    bad = _tokens(cfg.vocab, 2, cfg.seq_len, 2)
    bad[5] = cfg.vocab + 3
    with pytest.raises(IndexError, match="out of range"):
        s.train_step(bad, 2, step=1)
    _same_state(before, _state(s))
    # the session continues exactly like one that never saw the bad batch
    cfg2, t = _fresh()
    t.train_step(good, 2, step=0)
    nxt = _tokens(cfg.vocab, 2, cfg.seq_len, 3)
    assert s.train_step(nxt, 2, step=1) == t.train_step(nxt, 2, step=1)
    _same_state(_state(s), _state(t))


def test_nonfinite_activation_train_step_updates_nothing():
    cfg, s = _fresh()
    g = s.download("layers.1.ln2_g")
    g[3] = np.inf
    s.upload("layers.1.ln2_g", g)
    before = _state(s)
    with pytest.raises(RuntimeError, match=r"non-finite value at rmsnorm2 \(layer 1\)"):
        s.train_step(_tokens(cfg.vocab, 2, cfg.seq_len, 4), 2, step=0)
    _same_state(before, _state(s))


def test_adamw_nonfinite_gradient_names_tensor_and_updates_nothing():
    cfg, s = _fresh()
    s.build_step_context()
    s.zero_grads()
    s.forward(_tokens(cfg.vocab, 2, cfg.seq_len, 6), 2)
    s.backward(0)
    before = _state(s)
    with pytest.raises(RuntimeError, match="adamw_step: non-finite gradient in embed"):
        s.adamw_step(float("inf"))
    _same_state(before, _state(s))
    s.adamw_step(1.0)  # still usable
