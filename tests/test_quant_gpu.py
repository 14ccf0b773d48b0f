"""Absmax + FP8 cast kernels vs the reference (bit-exact).

Reference: absmax src/numerics.cpp:141-148, absmax_scale :150-158,
quantize_with_absmax :160-176, transpose_quantize_with_absmax
src/tensorops.cpp:164-182; tests mirror tests/test_numerics.cpp:151-226 and
tests/test_tensorops.cpp:169-197.
"""
import numpy as np
import pytest

from tests.helpers import rng_floats

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)


@pytest.fixture(scope="module")
def ops():
    from paper_2512_15306_b200 import ops
    return ops


@pytest.mark.parametrize("n", [1, 7, 8, 1000, 4096 + 3, 1 << 20, 3 * (1 << 20) + 17])
def test_absmax_bitexact(ops, ref, n):
    x = rng_floats(n, n, -3.0, 3.0)
    x[n // 2] = -7.25
    slot = ops.absmax(_bf16(x))
    assert ops.amax_value(slot) == ref.absmax(x)


def test_absmax_nan_sticky(ops):
    x = rng_floats(1, 10000, -1, 1)
    x[1234] = np.nan
    slot = ops.absmax(_bf16(x))
    assert np.isnan(ops.amax_value(slot))


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("n", [16, 1000, 65536 + 5, 1 << 22])
def test_quantize_bitexact(ops, ref, kind, n):
    x = rng_floats(10 + n, n, -5.0, 5.0)
    xt = _bf16(x)
    slot = ops.absmax(xt)
    amax = ops.amax_value(slot)
    codes, scale = ops.quantize(xt, kind, slot)
    rc, rs = ref.quantize_with_absmax(x, kind, amax)
    assert scale.item() == rs
    np.testing.assert_array_equal(codes.cpu().numpy(), rc)


@pytest.mark.parametrize("kind", [0, 1])
def test_quantize_worked_example(ops, kind):
    # tests/test_numerics.cpp:169-186: [1,-2,4] -> scale fmax/4, codes of 112/-224/448 (E4M3)
    x = np.array([1.0, -2.0, 4.0], np.float32)
    xt = _bf16(x)
    slot = ops.absmax(xt)
    codes, scale = ops.quantize(xt, kind, slot)
    fmax = 448.0 if kind == 0 else 57344.0
    assert scale.item() == fmax / 4
    from oracle import ref as R
    if R.available():
        np.testing.assert_array_equal(codes.cpu().numpy(), R.quantize_with_absmax(x, kind, 4.0)[0])


@pytest.mark.parametrize("kind", [0, 1])
def test_encode_all_bf16_patterns(ops, ref, kind):
    """Every bf16 bit pattern (incl. denormals, inf, NaN) through the device
    encoder with scale 1 vs the reference table encoder."""
    bits = np.arange(65536, dtype=np.uint32) << 16
    x = bits.view(np.float32)
    xt = torch.from_numpy(np.arange(65536, dtype=np.int32).astype(np.int16)).cuda().view(torch.bfloat16)
    fmax = 448.0 if kind == 0 else 57344.0
    slot = torch.tensor([np.float32(fmax).view(np.int32)], dtype=torch.int32, device="cuda")
    codes, scale = ops.quantize(xt, kind, slot)
    assert scale.item() == 1.0
    clamped = np.clip(x, -fmax, fmax)  # quantize_with_absmax clamps before encoding (numerics.cpp:172)
    want = ref.f8_encode(clamped, kind)
    got = codes.cpu().numpy()
    finite = ~np.isnan(x)
    np.testing.assert_array_equal(got[finite], want[finite])
    assert np.all((got[~finite] & 0x7F) == 0x7F)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("shape", [(64, 64), (100, 37), (256, 896), (1024, 136), (3, 5)])
def test_transpose_quantize_bitexact(ops, ref, kind, shape):
    r, c = shape
    x = rng_floats(r * 1000 + c, r * c, -2.0, 2.0).reshape(r, c)
    xt = _bf16(x)
    slot = ops.absmax(xt)
    amax = ops.amax_value(slot)
    ct, crm, scale = ops.quantize_transpose(xt, kind, slot, with_rowmajor=True)
    want_t, ws = ref.transpose_quantize_with_absmax(x, kind, amax)
    want_rm, _ = ref.quantize_with_absmax(x, kind, amax)
    assert scale.item() == ws
    np.testing.assert_array_equal(ct.cpu().numpy(), want_t)
    np.testing.assert_array_equal(crm.cpu().numpy(), want_rm)
