"""Per-op parity of the fused block kernels against the reference primitives on
identical inputs (teacher-forced: no FP8 chaos upstream).

  rmsnorm_residual_fused / _backward   src/tensorops.cpp:61-112  -> bit-exact values and absmax;
                                        dgamma: fixed-order two-level sum (<= 1e-6 rel)
  swiglu_fused / _backward             src/tensorops.cpp:114-153 -> <= 1 bf16 ulp (expf vs glibc)
  rope_apply                           src/model.cpp:171-191     -> bit-exact (host cos/sin table)
  sdpa_chunked / _backward             src/tensorops.cpp:191-303 -> <= 1 bf16 ulp on >= 99 %
  fused_cross_entropy_chunked          src/tensorops.cpp:344-410 -> loss <= 1e-5 rel, grads <= 1e-4
"""
import numpy as np
import pytest

from tests.helpers import bf16_grid_round, rng_floats

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2512_15306_b200 import ops
    return ops


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)


def _np(t):
    return t.float().cpu().numpy()


def _ulp(a, b):
    ai = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64) >> 16
    bi = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64) >> 16
    return np.abs(ai - bi)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("rows,d", [(1, 64), (37, 256), (300, 896), (64, 4096), (200, 4096), (96, 5120)])
@pytest.mark.parametrize("with_x", [False, True])
def test_rmsnorm_fwd_bitexact(ops, ref, rows, d, with_x):
    res = rng_floats(rows + d, rows * d, -3, 3).reshape(rows, d)
    x = rng_floats(rows * 3 + d, rows * d, -1, 1).reshape(rows, d) if with_x else None
    gamma = bf16_grid_round(rng_floats(7, d, 0.5, 1.5))
    nr_w, normed_w, am_w = ref.rmsnorm_residual_fused(x, res, gamma)
    nr, normed, slot = ops.rmsnorm_fwd(_bf16(x) if with_x else None, _bf16(res), _bf16(gamma))
    np.testing.assert_array_equal(_np(normed), normed_w)
    if with_x:
        np.testing.assert_array_equal(_np(nr), nr_w)
    assert ops.amax_value(slot) == am_w


@pytest.mark.parametrize("rows,d", [(5, 64), (300, 896), (40, 2048), (200, 4096), (96, 5120)])
@pytest.mark.parametrize("with_extra", [False, True])
def test_rmsnorm_bwd(ops, ref, rows, d, with_extra):
    nr = rng_floats(1 + d, rows * d, -3, 3).reshape(rows, d)
    dy = rng_floats(2 + d, rows * d, -1, 1).reshape(rows, d)
    ex = rng_floats(3 + d, rows * d, -1, 1).reshape(rows, d) if with_extra else None
    gamma = bf16_grid_round(rng_floats(4, d, 0.5, 1.5))
    din_w, dg_w = ref.rmsnorm_residual_backward(nr, gamma, dy, ex)
    din, dg, slot = ops.rmsnorm_bwd(_bf16(nr), _bf16(gamma), _bf16(dy), _bf16(ex) if with_extra else None)
    np.testing.assert_array_equal(_np(din), din_w)          # per-row sequential dot: bit-exact
    assert ops.amax_value(slot) == np.abs(din_w).max()
    assert _rel(dg.cpu().numpy(), dg_w) < 1e-6               # column sums: fixed but different order


@pytest.mark.parametrize("rows,h", [(3, 8), (256, 768), (100, 4864)])
def test_swiglu(ops, ref, rows, h):
    gu = rng_floats(rows + h, rows * 2 * h, -4, 4).reshape(rows, 2 * h)
    dh = rng_floats(rows + 2 * h, rows * h, -1, 1).reshape(rows, h)
    hw, am_w = ref.swiglu_fused(gu)
    hg, slot = ops.swiglu_fwd(_bf16(gu))
    d = _ulp(_np(hg), hw)
    assert d.max() <= 1 and (d == 0).mean() > 0.999
    dw = ref.swiglu_backward(gu, dh)
    dg, _ = ops.swiglu_bwd(_bf16(gu), _bf16(dh))
    d = _ulp(_np(dg), dw)
    assert d.max() <= 1 and (d == 0).mean() > 0.999


def test_swiglu_fast_quotient_exhaustive(ops):
    """The SwiGLU kernels' branch-free x/(1+e) and 1/(1+e) equal div.rn / rcp.rn
    on all 65536 bf16 gate values -- the quotient depends on nothing else, so
    the kernels' outputs are those of the div.rn formulation for every input."""
    from paper_2512_15306_b200 import _lib
    c = torch.zeros(6, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().qtk_swiglu_selfcheck(c.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "qtk_swiglu_selfcheck")
    bad_q, bad_s, fast, g_bits, q, q_ref = c.cpu().tolist()
    assert bad_q == 0 and bad_s == 0, (bad_q, bad_s, hex(g_bits), hex(q & 0xFFFFFFFF), hex(q_ref & 0xFFFFFFFF))
    assert fast > 35000                         # fast path: 2^-100 <= |g| <= 2^100 and 1+e <= 2^100


def test_swiglu_special_values(ops, ref):
    """Zeros of both signs, huge / tiny / subnormal gates (slow-path vectors) next to ordinary ones."""
    specials = np.array([0.0, -0.0, 1e-40, -1e-40, 1e-30, -100.0, -88.5, 90.0, 3e38, -3e38, 1.0, -1.0,
                         0.5, -0.5, 2.0, 7.0], np.float32)
    rows, h = 6, 16
    gu = rng_floats(11, rows * 2 * h, -4, 4).reshape(rows, 2 * h)
    gu[0, :h] = specials
    gu[3, :h] = specials[::-1]
    dh = rng_floats(12, rows * h, -1, 1).reshape(rows, h)
    gu = bf16_grid_round(gu)
    hw, _ = ref.swiglu_fused(gu)
    hg, _ = ops.swiglu_fwd(_bf16(gu))
    d = _ulp(_np(hg), hw)
    assert d.max() <= 1
    dw = ref.swiglu_backward(gu, dh)
    dg, _ = ops.swiglu_bwd(_bf16(gu), _bf16(dh))
    assert _ulp(_np(dg), dw).max() <= 1


def _qkv_np(B, T, H, Hkv, hd, seed):
    d = H * hd
    q = d + 2 * Hkv * hd
    return rng_floats(seed, B * T * q, -1.5, 1.5).reshape(B * T, q)


def _split(qkv, b, T, H, Hkv, hd):
    d = H * hd
    rows = qkv[b * T:(b + 1) * T]
    q3 = rows[:, :d].reshape(T, H, hd).transpose(1, 0, 2)
    k3 = rows[:, d:d + Hkv * hd].reshape(T, Hkv, hd).transpose(1, 0, 2)
    v3 = rows[:, d + Hkv * hd:].reshape(T, Hkv, hd).transpose(1, 0, 2)
    return q3, k3, v3


ATT_SHAPES = [(1, 64, 2, 1, 64), (2, 256, 4, 4, 64), (1, 200, 4, 2, 64), (1, 256, 2, 1, 128), (2, 96, 4, 1, 32)]


@pytest.mark.parametrize("B,T,H,Hkv,hd", ATT_SHAPES)
def test_attention_fwd(ops, ref, B, T, H, Hkv, hd):
    qkv = _qkv_np(B, T, H, Hkv, hd, T + hd)
    out, out32, lse, slot = ops.attn_fwd(_bf16(qkv), B, T, H, Hkv, hd)
    got = _np(out)
    want = np.concatenate([ref.sdpa(*_split(qkv, b, T, H, Hkv, hd)).transpose(1, 0, 2).reshape(T, H * hd)
                           for b in range(B)])
    # sum_j p_j |v_j|: the scale of the f32 rounding noise where sum_j p_j v_j cancels
    absq = np.abs(qkv)
    scale = np.concatenate([ref.sdpa(_split(qkv, b, T, H, Hkv, hd)[0], _split(qkv, b, T, H, Hkv, hd)[1],
                                     _split(absq, b, T, H, Hkv, hd)[2]).transpose(1, 0, 2).reshape(T, H * hd)
                            for b in range(B)])
    d = _ulp(got, want)
    bad = (d > 1) & (np.abs(got - want) > 1e-5 * scale)
    assert not bad.any(), (bad.sum(), d.max())
    assert (d == 0).mean() > 0.99, (d == 0).mean()
    assert ops.amax_value(slot) == np.abs(got).max()


@pytest.mark.parametrize("B,T,H,Hkv,hd", ATT_SHAPES)
def test_attention_bwd(ops, ref, B, T, H, Hkv, hd):
    qkv = _qkv_np(B, T, H, Hkv, hd, 3 * T + hd)
    d = H * hd
    go = rng_floats(5 * T + hd, B * T * d, -1, 1).reshape(B * T, d)
    qt = _bf16(qkv)
    out, out32, lse, _ = ops.attn_fwd(qt, B, T, H, Hkv, hd)
    dqkv = _np(ops.attn_bwd(qt, out32, _bf16(go), lse, B, T, H, Hkv, hd))
    for b in range(B):
        q3, k3, v3 = _split(qkv, b, T, H, Hkv, hd)
        go3 = go[b * T:(b + 1) * T].reshape(T, H, hd).transpose(1, 0, 2)
        dq, dk, dv = ref.sdpa_backward(q3, k3, v3, go3)
        g = dqkv[b * T:(b + 1) * T]
        gq = g[:, :d].reshape(T, H, hd).transpose(1, 0, 2)
        gk = g[:, d:d + Hkv * hd].reshape(T, Hkv, hd).transpose(1, 0, 2)
        gv = g[:, d + Hkv * hd:].reshape(T, Hkv, hd).transpose(1, 0, 2)
        for name, x, y in (("dq", gq, dq), ("dk", gk, dk), ("dv", gv, dv)):
            r = _rel(x, y)
            assert r < 2e-3, (name, r)
            assert (_ulp(x, y) <= 1).mean() > 0.99, name


@pytest.mark.parametrize("rows,T,H,hd", [(128, 64, 2, 64), (512, 256, 4, 64), (256, 128, 2, 128)])
def test_rope_bitexact(ops, ref, rows, T, H, hd):
    """RoPE fwd + bwd (src/model.cpp:171-191) vs a numpy restatement on the
    same float32 table the reference computes."""
    import ctypes
    Hkv = 1
    q = H * hd + 2 * Hkv * hd
    x = rng_floats(rows + hd, rows * q, -2, 2).reshape(rows, q)
    half = hd // 2
    i = np.arange(half, dtype=np.float32)
    freq = np.power(np.float32(10000.0), (np.float32(-2.0) * i / np.float32(hd)).astype(np.float32)).astype(np.float32)
    t = (np.arange(rows) % T).astype(np.float32)
    ang = (t[:, None] * freq[None, :]).astype(np.float32)
    cs, sn = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
    tab = torch.from_numpy(np.stack([cs[:T], sn[:T]], -1).astype(np.float32).copy()).cuda()
    for bwd in (0, 1):
        want = x.copy()
        s = -sn if bwd else sn
        for h in range(H + Hkv):
            a = x[:, h * hd:h * hd + half]
            b = x[:, h * hd + half:(h + 1) * hd]
            want[:, h * hd:h * hd + half] = bf16_grid_round((a * cs - b * s).astype(np.float32))
            want[:, h * hd + half:(h + 1) * hd] = bf16_grid_round((a * s + b * cs).astype(np.float32))
        xt = _bf16(x)
        from paper_2512_15306_b200 import _lib
        am = torch.zeros(1, dtype=torch.int32, device="cuda")
        rc = _lib.lib().qtk_rope(xt.data_ptr(), rows, T, H + Hkv, hd, q, tab.data_ptr(), bwd,
                                 am.data_ptr() if bwd else None, torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        np.testing.assert_array_equal(_np(xt), want)
        if bwd:  # absmax over the whole row, v columns included
            want_am = np.abs(bf16_grid_round(want)).max()
            assert am.view(torch.float32).item() == want_am


@pytest.mark.parametrize("N,d,V", [(128, 128, 256), (300, 256, 1000), (64, 896, 4096)])
def test_cross_entropy(ops, ref, N, d, V):
    h = rng_floats(N + d, N * d, -1, 1).reshape(N, d)
    w = rng_floats(V + d, V * d, -0.2, 0.2).reshape(V, d)
    t = np.random.default_rng(N).integers(0, V, N).astype(np.int32)
    loss, dh, dw = ref.cross_entropy(h, w, t)
    H, W = _bf16(h), _bf16(w)
    logits = ops.gemm(H, W, M=N, N=V, K=d, epi=ops.EPI_F32)
    lr, hi, lo = ops.ce_softmax(logits, torch.from_numpy(t).cuda(), 1.0 / N)
    assert abs(lr.sum().item() / N - loss) / loss < 1e-5, (lr.sum().item() / N, loss)
    dh_g = ops.gemm(hi, W, M=N, N=d, K=V, b_mn=True, epi=ops.EPI_BF16, a2=lo)
    d_ = _ulp(_np(dh_g), dh)
    assert (d_ == 0).mean() > 0.99, (d_ == 0).mean()
    assert _rel(_np(dh_g), dh) < 1e-3
    dw_g = ops.gemm(hi, H, M=V, N=d, K=N, a_mn=True, b_mn=True, epi=ops.EPI_F32, a2=lo)
    assert _rel(dw_g.cpu().numpy(), dw) < 1e-4


@pytest.mark.parametrize("N,d,V", [(256, 128, 1000), (300, 256, 4100)])
def test_ce_stats_epilogue_matches_two_pass(ops, N, d, V):
    """Logits GEMM with the softmax-statistics epilogue + single-pass CE equals the
    two-pass CE kernel on the same logits (loss 1e-6 rel; dlogits hi bit-exact on
    >= 99.9 %; hi + lo within 5e-5: the block statistics use ex2 and a different
    summation grouping, ~1e-6 on the denominator, amplified on single elements by
    the bf16 rounding of lo)."""
    g = torch.Generator(device="cpu").manual_seed(3)
    h = (torch.randn(N, d, generator=g) * 0.5).to(torch.bfloat16).cuda()
    w = (torch.randn(V, d, generator=g) * 0.5).to(torch.bfloat16).cuda()
    t = torch.randint(0, V, (N,), generator=g, dtype=torch.int32).cuda()
    stats = torch.empty(N, (V + 127) // 128, 2, dtype=torch.float32, device="cuda")
    tl = torch.empty(N, dtype=torch.float32, device="cuda")
    logits = ops.gemm(h, w, M=N, N=V, K=d, epi=ops.EPI_F32, ce=(t, stats, tl))
    l2, hi2, lo2 = ops.ce_softmax(logits, t, 1.0 / N)
    l1, hi1, lo1 = ops.ce_softmax_stats(logits, t, stats, tl, 1.0 / N)
    torch.cuda.synchronize()
    assert torch.allclose(l1, l2, rtol=1e-6, atol=1e-6)
    assert torch.equal(tl, logits[torch.arange(N), t.long()])
    same = (hi1.view(torch.int16) == hi2.view(torch.int16)).float().mean().item()
    assert same >= 0.999, same
    full1 = hi1.float() + lo1.float()
    full2 = hi2.float() + lo2.float()
    assert torch.allclose(full1, full2, rtol=5e-5, atol=1e-12)


@pytest.mark.parametrize("B,T,H,Hkv,hd", [(2, 256, 4, 2, 64), (1, 384, 4, 1, 64), (2, 200, 4, 4, 128),
                                          (4, 1024, 14, 2, 64), (2, 1024, 32, 32, 128), (3, 640, 8, 2, 128)])
def test_attention_fwd_two_tile_kernel_bitwise_equals_one_tile(ops, B, T, H, Hkv, hd):
    """fwd2q_tc_kernel (two query tiles per CTA, P through TMEM) reproduces fwd1p_tc_kernel
    bit for bit (out, unrounded out32, LSE, absmax): same P operands, same PV issue order,
    l summed per key half as the one-tile kernel's two half-row threads do.  Odd tile
    counts and ragged T included."""
    from paper_2512_15306_b200 import _lib
    L = _lib.lib()
    d = H * hd
    q = d + 2 * Hkv * hd
    g = torch.Generator(device="cuda").manual_seed(T + hd)
    qkv = (torch.randn(B * T, q, device="cuda", generator=g) * 1.5).to(torch.bfloat16)
    res = []
    try:
        for mode in (0, 1):
            L.qtk_attn_set_fwd2q(mode)
            res.append(ops.attn_fwd(qkv, B, T, H, Hkv, hd))
    finally:
        L.qtk_attn_set_fwd2q(1)
    for a, b in zip(*res):
        assert torch.equal(a, b)


@pytest.mark.parametrize("rows,d,resid", [(16384, 896, True), (200, 896, True), (8192, 4096, True), (300, 4096, False),
                                          (77, 5120, True), (1000, 1536, True)])
def test_rmsnorm_split_role_chain_bitwise(ops, rows, d, resid):
    """rms_chain2_kernel (producer warps form the terms, one chain lane per row adds them)
    gives the same inv / normed / nr / d_in / absmax as the fused single-pass kernels and the
    one-role chain kernel: the same f32 operations in the same order (dgamma: same partials
    only when both runs take the chain + rows path; against the fused path's coarser partials
    it is a regrouped sum, compared within 2e-4)."""
    from paper_2512_15306_b200 import _lib
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(rows + d)
    bf = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.7).to(torch.bfloat16)
    x, res, dy, ex, gam = bf(rows, d), bf(rows, d), bf(rows, d), bf(rows, d), bf(d) + 1
    outs = []
    try:
        for mode in (0, 1, 2, 3):
            L.qtk_rms_set_path(mode)
            nr, normed, s1 = ops.rmsnorm_fwd(x if resid else None, res, gam)
            din, dg, s2 = ops.rmsnorm_bwd(nr if resid else res, gam, dy, ex)
            torch.cuda.synchronize()
            outs.append((nr, normed, s1, din, s2, dg))
    finally:
        L.qtk_rms_set_path(3)
    for mode, o in ((1, outs[1]), (2, outs[2]), (3, outs[3])):
        for k in range(5):
            if outs[0][k] is None:
                continue
            assert torch.equal(outs[0][k], o[k]), (mode, k)
        if mode in (1, 3):  # same backward path (and dgamma partials) as mode 0
            assert torch.equal(o[5], outs[0][5])
        else:  # fused partials (R rows) vs 16-row partials: same sums, regrouped
            torch.testing.assert_close(o[5], outs[0][5], rtol=2e-4, atol=1e-6)


@pytest.mark.parametrize("rows,T,H,Hkv,hd", [(16384, 1024, 14, 2, 64), (8192, 1024, 32, 32, 128), (300, 100, 4, 1, 64)])
def test_rope_head_looped_kernel_bitwise(rows, T, H, Hkv, hd):
    """rope_heads_kernel (one table chunk per row, looped over the heads) equals the per-item
    kernel bit for bit, forward and backward (with the whole-row absmax)."""
    from paper_2512_15306_b200 import _lib
    L = _lib.lib()
    q = (H + 2 * Hkv) * hd
    g = torch.Generator(device="cuda").manual_seed(rows + hd)
    x = (torch.randn(rows, q, device="cuda", generator=g) * 2).to(torch.bfloat16)
    tab = torch.randn(T, hd // 2, 2, device="cuda", generator=g)
    try:
        for bwd in (0, 1):
            outs = []
            for mode in (0, 1):
                L.qtk_rope_set_heads(mode)
                xt = x.clone()
                am = torch.zeros(1, dtype=torch.int32, device="cuda")
                rc = L.qtk_rope(xt.data_ptr(), rows, T, H + Hkv, hd, q, tab.data_ptr(), bwd,
                                am.data_ptr() if bwd else None, torch.cuda.current_stream().cuda_stream)
                assert rc == 0
                outs.append((xt, am))
            assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    finally:
        L.qtk_rope_set_heads(1)
