"""The C restatement (oracle/qtrain_oracle.c) pinned against the golden
vectors (tests/golden, identical to the reference's proj/data) and -- bit for
bit -- against the unmodified reference compiled from its sources
(oracle/_ref).  Mirrors tests/test_numerics.cpp and tests/test_tensorops.cpp
of the reference.  CPU only."""
import math
import pathlib
import struct

import numpy as np
import pytest

from tests.helpers import bf16_grid_round, rng_floats

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def port():
    from oracle import port as P
    if not P.available():
        pytest.skip("oracle/_build/liboracle.so not built")
    return P


def _golden_table(name):
    vals = []
    for line in (GOLD / name).read_text().splitlines():
        if line.startswith("#"):
            continue
        code, v = line.split()
        vals.append((int(code, 16), float(v)))
    return vals


@pytest.mark.parametrize("kind,name", [(0, "fp8_e4m3_test_vectors.txt"), (1, "fp8_e5m2_test_vectors.txt")])
def test_decode_matches_golden(port, kind, name):
    tab = port.f8_decode_table(kind)
    for code, v in _golden_table(name):
        if math.isnan(v):
            assert math.isnan(tab[code])
        else:
            assert tab[code] == v, (code, tab[code], v)


def test_fmax(port):
    assert port.lib().qto_f8_fmax(0) == 448.0 and port.lib().qto_f8_fmax(1) == 57344.0


def test_rng_matches_golden(port):
    for line in (GOLD / "rng_test_vectors.txt").read_text().splitlines():
        if line.startswith("#"):
            continue
        s, t, c, want = map(int, line.split())
        assert port.rng_uniform(s, t, c) == want


def _u2f(u):
    return struct.unpack("<f", struct.pack("<I", u))[0]


def _f2u(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def test_bf16_and_sr_golden(port):
    for line in (GOLD / "bf16_round_vectors.txt").read_text().splitlines()[1:]:
        x, r = (int(v, 16) for v in line.split())
        assert _f2u(port.bf16_round(_u2f(x))) == r
    for line in (GOLD / "sr_vectors.txt").read_text().splitlines()[1:]:
        x, seed, stream, ctr, r = line.split()
        assert _f2u(port.stochastic_round_bf16(_u2f(int(x, 16)), int(seed), int(stream), int(ctr))) == int(r, 16)


def test_worked_example(port):
    # tests/test_numerics.cpp:169-186
    codes, s = port.quantize_with_absmax(np.array([1, -2, 4], np.float32), 0, 4.0)
    assert s == 112.0
    tab = port.f8_decode_table(0)
    assert [tab[c] for c in codes] == [112.0, -224.0, 448.0]


@pytest.mark.parametrize("kind", [0, 1])
def test_encode_is_rne_nearest(port, kind):
    """Brute-force nearest representable with ties to the even code
    (tests/test_numerics.cpp:118-149)."""
    tab = port.f8_decode_table(kind)
    fin = [(v, c) for c, v in enumerate(tab[:128]) if np.isfinite(v)]
    vals = np.array([v for v, _ in fin], np.float64)
    codes = [c for _, c in fin]
    fmax = vals.max()
    x = np.random.default_rng(kind).uniform(-1.2 * fmax, 1.2 * fmax, 4000).astype(np.float32)
    x = np.concatenate([x, (vals[:-1] + vals[1:]).astype(np.float32) / 2])  # exact midpoints
    got = port.f8_encode(x, kind)
    for xi, gi in zip(x, got):
        a = min(abs(float(xi)), fmax)
        d = np.abs(vals - a)
        best = np.flatnonzero(d == d.min())
        cs = [codes[i] for i in best]
        want = cs[0] if len(cs) == 1 else [c for c in cs if c % 2 == 0][0]
        if xi < 0 or (xi == 0 and math.copysign(1, xi) < 0):
            want |= 0x80
        assert gi == want, (xi, gi, want)


# ---------------------------------------------------------------------------
# restatement == reference, bit for bit
# ---------------------------------------------------------------------------
def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint32) if a.dtype == np.float32 else a,
                          b.view(np.uint32) if b.dtype == np.float32 else b)


@pytest.mark.parametrize("kind", [0, 1])
def test_encode_all_bf16_patterns_vs_reference(port, ref, kind):
    x = (np.arange(65536, dtype=np.uint32) << 16).view(np.float32)
    _eq(port.f8_encode(x, kind), ref.f8_encode(x, kind))


@pytest.mark.parametrize("kind", [0, 1])
def test_quantize_vs_reference(port, ref, kind):
    x = rng_floats(3 + kind, 5000, -7, 7)
    a = ref.absmax(x)
    assert port.absmax(x) == a
    assert port.absmax_scale(a, kind) == ref.absmax_scale(a, kind)
    c1, s1 = port.quantize_with_absmax(x, kind, a)
    c2, s2 = ref.quantize_with_absmax(x, kind, a)
    assert s1 == s2
    _eq(c1, c2)
    m = x[:4000].reshape(40, 100)
    _eq(port.transpose_quantize_with_absmax(m, kind, a)[0], ref.transpose_quantize_with_absmax(m, kind, a)[0])


def test_absmax_nan_raises(port):
    x = np.ones(10, np.float32)
    x[3] = np.nan
    with pytest.raises(RuntimeError, match="NaN"):
        port.absmax(x)


def test_matmul_vs_reference(port, ref):
    a = rng_floats(1, 48 * 96, -1, 1).reshape(48, 96)
    b = rng_floats(2, 40 * 96, -1, 1).reshape(40, 96)
    ac, sa = port.quantize_with_absmax(a, 1, port.absmax(a))
    bc, sb = port.quantize_with_absmax(b, 0, port.absmax(b))
    _eq(port.matmul_fp8(ac, 1, sa, bc, 0, sb), ref.matmul_fp8(ac, 1, sa, bc, 0, sb))
    _eq(port.matmul_f32(a, b), ref.matmul_f32(a, b))


def test_fused_ops_vs_reference(port, ref):
    rows, d = 17, 96
    res = rng_floats(5, rows * d, -3, 3).reshape(rows, d)
    x = rng_floats(6, rows * d, -1, 1).reshape(rows, d)
    g = bf16_grid_round(rng_floats(7, d, 0.5, 1.5))
    for xx in (None, x):
        a, b = port.rmsnorm_residual_fused(xx, res, g), ref.rmsnorm_residual_fused(xx, res, g)
        _eq(a[0], b[0])
        _eq(a[1], b[1])
        assert a[2] == b[2]
    dy = rng_floats(8, rows * d, -1, 1).reshape(rows, d)
    for ex in (None, x):
        a, b = port.rmsnorm_residual_backward(res, g, dy, ex), ref.rmsnorm_residual_backward(res, g, dy, ex)
        _eq(a[0], b[0])
        _eq(a[1], b[1])
    gu = rng_floats(9, rows * 64, -4, 4).reshape(rows, 64)
    dh = rng_floats(10, rows * 32, -1, 1).reshape(rows, 32)
    _eq(port.swiglu_fused(gu)[0], ref.swiglu_fused(gu)[0])
    _eq(port.swiglu_backward(gu, dh), ref.swiglu_backward(gu, dh))


def test_sdpa_vs_reference(port, ref):
    H, Hkv, T, D = 4, 2, 20, 16
    q = rng_floats(11, H * T * D, -1, 1).reshape(H, T, D)
    k = rng_floats(12, Hkv * T * D, -1, 1).reshape(Hkv, T, D)
    v = rng_floats(13, Hkv * T * D, -1, 1).reshape(Hkv, T, D)
    go = rng_floats(14, H * T * D, -1, 1).reshape(H, T, D)
    _eq(port.sdpa(q, k, v), ref.sdpa(q, k, v, chunk_rows=7))  # chunk-invariant (tests/test_tensorops.cpp:246-261)
    for a, b in zip(port.sdpa_backward(q, k, v, go), ref.sdpa_backward(q, k, v, go, chunk_rows=3)):
        _eq(a, b)


def test_embedding_and_ce_vs_reference(port, ref):
    ids = np.random.default_rng(3).integers(0, 11, 50).astype(np.int32)
    go = rng_floats(15, 50 * 8, -1, 1).reshape(50, 8)
    _eq(port.embedding_backward(ids, go, 11), ref.embedding_backward(ids, go, 11))
    with pytest.raises(IndexError):
        port.embedding_backward(np.array([11], np.int32), go[:1], 11)
    h = rng_floats(16, 30 * 24, -1, 1).reshape(30, 24)
    w = rng_floats(17, 40 * 24, -1, 1).reshape(40, 24)
    t = np.random.default_rng(4).integers(0, 40, 30).astype(np.int32)
    a, b = port.cross_entropy(h, w, t), ref.cross_entropy(h, w, t, chunk=7)
    assert a[0] == b[0]
    _eq(a[1], b[1])
    _eq(a[2], b[2])


@pytest.mark.parametrize("bf16_moments", [False, True])
def test_adamw_norm_accumulate_vs_reference(port, ref, bf16_moments):
    n = 1000
    p = bf16_grid_round(rng_floats(20, n, -1, 1))
    m = rng_floats(21, n, -1e-2, 1e-2)
    v = rng_floats(22, n, 0, 1e-3)
    g = bf16_grid_round(rng_floats(23, n, -1, 1))
    for step in (0, 5):
        a = port.adamw_tensor("layers.3.w_o", p, m, v, g, lr=3e-3, wd=0.1, bf16_moments=bf16_moments, seed=9,
                              step_count=step, grad_scale=0.25)
        b = ref.adamw_tensor("layers.3.w_o", p, m, v, g, lr=3e-3, wd=0.1, bf16_moments=bf16_moments, seed=9,
                             step_count=step, grad_scale=0.25)
        for x, y in zip(a, b):
            _eq(x, y)
    assert port.grad_norm_partials(g) == ref.grad_norm_partials(g)
    _eq(port.grad_accumulate("embed", m, g, seed=4, micro_step=3), ref.grad_accumulate("embed", m, g, seed=4,
                                                                                          micro_step=3))


def test_init_normal_vs_reference(port, ref):
    rm = ref.RefModel([1, 32, 64, 2, 1, 16, 8], 1234)
    std = 1.0 / math.sqrt(32.0)
    std = float(np.float32(1.0) / np.sqrt(np.float32(32.0)))
    for name in ("embed", "layers.0.w_qkv", "lm_head"):
        want = rm.get(name)
        _eq(port.init_normal(want.size, std, 1234, name), want)


def test_zero1_sharded_adamw_is_bitwise_unsharded(port):
    """ZeRO-1 with global-index RNG keys == unsharded (tests/test_optim.cpp:155-181)."""
    for n, W in ((1000, 2), (3000, 4), (255, 8)):
        p = bf16_grid_round(rng_floats(30 + W, n, -1, 1))
        g = bf16_grid_round(rng_floats(31 + W, n, -1, 1))
        z = np.zeros(n, np.float32)
        full = port.adamw_tensor("w", p, z, z, g, seed=1)[0]
        padded, pw = port.shard_layout(n, W)
        assert padded % (256 * W) == 0 and pw * W == padded
        out = p.copy()
        for w in range(W):
            lo, hi = min(w * pw, n), min((w + 1) * pw, n)
            if lo < hi:
                part = port.adamw_tensor("w", p, z, z, g, seed=1, lo=lo, hi=hi)[0]
                out[lo:hi] = part[lo:hi]
        _eq(out, full)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_reference_reduce_scatter_protocol_equals_oracle(ref, W):
    """The reference's copy-engine protocol (src/comms.cpp:185-229) and its
    straight-summation oracle (:233-254) agree bitwise (SR and f32 modes) -- the
    contract qtk_reduce_scatter_sr is checked against on the GPU."""
    n = 1000
    chunks = bf16_grid_round(rng_floats(70 + W, W * W * n, -1, 1)).reshape(W, W, n)
    acc = bf16_grid_round(rng_floats(80 + W, W * n, -0.5, 0.5)).reshape(W, n)
    for sto in (True, False):
        a = ref.reduce_scatter(chunks, acc, stochastic=sto, seed=9, step=3, layer=1)
        b = ref.reduce_scatter(chunks, acc, stochastic=sto, seed=9, step=3, layer=1, protocol=True)
        np.testing.assert_array_equal(a, b)
