"""tcgen05 GEMM vs the reference matmul_tn (src/tensorops.cpp:24-59).

FP8 outputs: the oracle accumulates sequentially in f32, the tensor core in a
different order, so outputs are compared at <=1 bf16 ulp on >=99.9 % of
elements (calibrated by Appendix P5: the oracle itself sits 1
ulp from exact on 0.01-0.02 % of outputs).  Layout flags (K- vs MN-major
operands) must not change a single bit.
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


def _q(ref, x, kind):
    amax = ref.absmax(x)
    codes, s = ref.quantize_with_absmax(x, kind, amax)
    return codes, s


def _cuda_u8(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint8)).cuda()


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)


def _ulp_diff(a, b):
    ai = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64) >> 16
    bi = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64) >> 16
    return np.abs(ai - bi)


def _check_close(got, want, frac=0.999, absscale=None, K=1):
    """<=1 bf16 ulp, except where the sum cancels: there the f32 ordering error
    of the oracle itself (~sqrt(K) eps_f32 sum|a_k b_k|) dominates the ulp of
    the small result, so allow that much absolute error."""
    d = _ulp_diff(got, want)
    bad = d > 1
    if absscale is not None and bad.any():
        tol = 8.0 * np.sqrt(K) * 2.0 ** -24 * absscale
        bad &= np.abs(got.astype(np.float64) - want) > tol
    assert not bad.any(), f"{bad.sum()} elements beyond tolerance (max ulp diff {d.max()})"
    assert (d == 0).mean() >= frac, f"only {(d == 0).mean():.5f} exact"


def _absscale(ref, ac, ak, sa, bc, bk, sb):
    ta, tb = ref.f8_decode_table(ak).astype(np.float64), ref.f8_decode_table(bk).astype(np.float64)
    return (np.abs(ta[ac]) @ np.abs(tb[bc]).T) / (np.float32(sa) * np.float32(sb))


SHAPES = [(128, 256, 128), (256, 1152, 896), (208, 304, 160), (144, 144, 96), (512, 512, 4864), (32, 64, 32)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("layout", ["kk", "kmn", "mnmn"])
@pytest.mark.parametrize("kinds", [(0, 0), (1, 0)])
def test_fp8_gemm_layouts(ops, ref, M, N, K, layout, kinds):
    ak, bk = kinds
    a = rng_floats(M * 7 + K, M * K, -1, 1).reshape(M, K)
    b = rng_floats(N * 13 + K, N * K, -0.5, 0.5).reshape(N, K)
    ac, sa = _q(ref, a, ak)
    bc, sb = _q(ref, b, bk)
    want = ref.matmul_fp8(ac, ak, sa, bc, bk, sb)
    A = _cuda_u8(ac if layout == "kk" or layout == "kmn" else ac.T.copy())
    B = _cuda_u8(bc if layout == "kk" else bc.T.copy())
    sa_t = torch.tensor([sa], dtype=torch.float32, device="cuda")
    sb_t = torch.tensor([sb], dtype=torch.float32, device="cuda")
    got = ops.gemm(A, B, M=M, N=N, K=K, a_mn=(layout == "mnmn"), b_mn=(layout != "kk"), a_fmt=ak, b_fmt=bk,
                   a_scale=sa_t, b_scale=sb_t, epi=ops.EPI_BF16)
    _check_close(got.float().cpu().numpy(), want, absscale=_absscale(ref, ac, ak, sa, bc, bk, sb), K=K)


@pytest.mark.parametrize("bn", [128, 256])
def test_fp8_gemm_bn_invariant(ops, ref, bn):
    M, N, K = 384, 640, 512
    a = rng_floats(1, M * K, -1, 1).reshape(M, K)
    b = rng_floats(2, N * K, -1, 1).reshape(N, K)
    ac, sa = _q(ref, a, 0)
    bc, sb = _q(ref, b, 0)
    sa_t = torch.tensor([sa], device="cuda")
    sb_t = torch.tensor([sb], device="cuda")
    g1 = ops.gemm(_cuda_u8(ac), _cuda_u8(bc), M=M, N=N, K=K, a_scale=sa_t, b_scale=sb_t, bn=bn)
    g2 = ops.gemm(_cuda_u8(ac.T.copy()), _cuda_u8(bc.T.copy()), M=M, N=N, K=K, a_mn=True, b_mn=True,
                  a_scale=sa_t, b_scale=sb_t, bn=bn)
    assert torch.equal(g1, g2)


def test_fp8_gemm_long_k_accuracy(ops, ref):
    """K=16384: tcgen05 f32 accumulation must stay within 1 bf16 ulp of the
    oracle (SURVEY.md §7 hard part 2)."""
    M, N, K = 128, 128, 16384
    a = rng_floats(5, M * K, -1, 1).reshape(M, K)
    b = rng_floats(6, N * K, -1, 1).reshape(N, K)
    ac, sa = _q(ref, a, 1)
    bc, sb = _q(ref, b, 0)
    want = ref.matmul_fp8(ac, 1, sa, bc, 0, sb)
    got = ops.gemm(_cuda_u8(ac), _cuda_u8(bc), M=M, N=N, K=K, a_fmt=1, b_fmt=0,
                   a_scale=torch.tensor([sa], device="cuda"), b_scale=torch.tensor([sb], device="cuda"))
    _check_close(got.float().cpu().numpy(), want, frac=0.995, absscale=_absscale(ref, ac, 1, sa, bc, 0, sb), K=K)


def test_fp8_gemm_residual_epilogue(ops, ref):
    M, N, K = 256, 384, 256
    a = rng_floats(11, M * K, -1, 1).reshape(M, K)
    b = rng_floats(12, N * K, -1, 1).reshape(N, K)
    r = rng_floats(13, M * N, -4, 4).reshape(M, N)
    ac, sa = _q(ref, a, 0)
    bc, sb = _q(ref, b, 0)
    lin = ref.matmul_fp8(ac, 0, sa, bc, 0, sb)           # bf16-rounded linear output
    want = bf16_grid_round(lin + r)                        # r_out = bf16(ffn_out + r_mid), model.cpp:281-283
    got = ops.gemm(_cuda_u8(ac), _cuda_u8(bc), M=M, N=N, K=K, a_scale=torch.tensor([sa], device="cuda"),
                   b_scale=torch.tensor([sb], device="cuda"), epi=ops.EPI_BF16_RES, res=_bf16(r))
    _check_close(got.float().cpu().numpy(), want, absscale=_absscale(ref, ac, 0, sa, bc, 0, sb) + np.abs(r), K=K)


def test_fp8_gemm_sr_accumulate_epilogue(ops, ref):
    """wgrad epilogue = GradAccumulator::accumulate (src/model.cpp:455-462)."""
    M, N, K = 256, 256, 1024
    a = rng_floats(21, M * K, -1, 1).reshape(M, K)
    b = rng_floats(22, N * K, -1, 1).reshape(N, K)
    ac, sa = _q(ref, a, 1)
    bc, sb = _q(ref, b, 0)
    g = ref.matmul_fp8(ac, 1, sa, bc, 0, sb)
    buf0 = rng_floats(23, M * N, -0.1, 0.1).reshape(M, N)
    seed, name, micro = 1234, "layers.0.w_o", 3
    want = ref.grad_accumulate(name, buf0, g, seed=seed, micro_step=micro)
    stream = ref.fnv1a64("gradaccum/" + name)
    buf = _bf16(buf0)
    ops.gemm(_cuda_u8(ac.T.copy()), _cuda_u8(bc.T.copy()), M=M, N=N, K=K, a_mn=True, b_mn=True, a_fmt=1, b_fmt=0,
             a_scale=torch.tensor([sa], device="cuda"), b_scale=torch.tensor([sb], device="cuda"),
             epi=ops.EPI_BF16_ACC, out=buf, sr=(seed, stream, micro * M * N))
    d = _ulp_diff(buf.float().cpu().numpy(), want)
    assert d.max() <= 1 and (d == 0).mean() >= 0.999


@pytest.mark.parametrize("layout", ["kk", "kmn", "mnmn"])
@pytest.mark.parametrize("M,N,K", [(128, 512, 64), (256, 304, 200), (384, 1024, 512)])
def test_bf16_gemm_f32_out(ops, ref, layout, M, N, K):
    a = rng_floats(31 + M, M * K, -1, 1).reshape(M, K)
    b = rng_floats(32 + N, N * K, -1, 1).reshape(N, K)
    want = ref.matmul_f32(a, b, round_bf16=False)
    A = _bf16(a if layout != "mnmn" else a.T.copy())
    B = _bf16(b if layout == "kk" else b.T.copy())
    got = ops.gemm(A, B, M=M, N=N, K=K, a_mn=(layout == "mnmn"), b_mn=(layout != "kk"), epi=ops.EPI_F32)
    g = got.cpu().numpy().astype(np.float64)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).T.astype(np.float64)
    assert (np.abs(g - want) <= 4.0 * np.sqrt(K) * 2.0 ** -24 * scale + 1e-30).all()


def test_bf16_gemm_bf16_out(ops, ref):
    M, N, K = 256, 896, 1024
    a = rng_floats(41, M * K, -1, 1).reshape(M, K)
    b = rng_floats(42, N * K, -1, 1).reshape(N, K)
    want = ref.matmul_f32(a, b, round_bf16=True)
    got = ops.gemm(_bf16(a), _bf16(b.T.copy()), M=M, N=N, K=K, b_mn=True, epi=ops.EPI_BF16)
    _check_close(got.float().cpu().numpy(), want, absscale=np.abs(a).astype(np.float64) @ np.abs(b).T, K=K)


def test_gemm_rejects_unaligned_stride(ops):
    """TMA needs 16-B aligned row strides; the C-ABI reports invalid_argument."""
    a = torch.zeros((64, 40), dtype=torch.uint8, device="cuda")
    b = torch.zeros((40, 100), dtype=torch.uint8, device="cuda")  # MN-major B with a 100-B row stride
    with pytest.raises(RuntimeError, match="status 1"):
        ops.gemm(a, b, M=64, N=100, K=40, b_mn=True)


@pytest.mark.parametrize("M,N", [(896, 896), (1152, 896)])
def test_fp8_gemm_splitk_wgrad(ops, ref, M, N):
    """Weight-gradient shape (out, in, K = tokens) with too few tiles for 148 SMs:
    the automatic split-K path (fixed-order partial sums) stays within the same
    tolerance of the reference as the unsplit kernel."""
    K = 8192
    a = rng_floats(M + 1, M * K, -1, 1).reshape(M, K)
    b = rng_floats(N + 2, N * K, -1, 1).reshape(N, K)
    ac, sa = _q(ref, a, 1)
    bc, sb = _q(ref, b, 0)
    want = ref.matmul_fp8(ac, 1, sa, bc, 0, sb)
    st = dict(M=M, N=N, K=K, a_mn=True, b_mn=True, a_fmt=1, b_fmt=0, a_scale=torch.tensor([sa], device="cuda"),
              b_scale=torch.tensor([sb], device="cuda"))
    A, B = _cuda_u8(ac.T.copy()), _cuda_u8(bc.T.copy())
    g_split = ops.gemm(A, B, split_k=0, **st)
    g_plain = ops.gemm(A, B, split_k=1, **st)
    scale = _absscale(ref, ac, 1, sa, bc, 0, sb)
    _check_close(g_split.float().cpu().numpy(), want, absscale=scale, K=K, frac=0.99)
    _check_close(g_plain.float().cpu().numpy(), want, absscale=scale, K=K, frac=0.99)


@pytest.mark.parametrize("M,H,K", [(256, 512, 256), (300, 1216, 384)])
def test_fp8_gemm_swiglu_backward_epilogue(ops, M, H, K):
    """Down-projection dgrad with swiglu_backward (src/tensorops.cpp:133-153) in the
    epilogue: bitwise equal to the separate dgrad (bf16 d_h) + SwiGLU-backward kernel,
    absmax included."""
    g = torch.Generator(device="cpu").manual_seed(5)
    ac = torch.randint(0, 120, (M, K), dtype=torch.uint8, generator=g).cuda()
    bc = torch.randint(0, 120, (H, K), dtype=torch.uint8, generator=g).cuda()  # W_down codes [d][Hh]: MN-major B
    bc = bc.t().contiguous()  # stored [K][N] for the (K,MN) dgrad layout
    gu = (torch.randn(M, 2 * H, generator=g) * 2).to(torch.bfloat16).cuda()
    sa, sb = torch.tensor([3.0], device="cuda"), torch.tensor([0.75], device="cuda")
    dh = ops.gemm(ac, bc, M=M, N=H, K=K, b_mn=True, a_scale=sa, b_scale=sb, epi=ops.EPI_BF16)
    want, slot = ops.swiglu_bwd(gu, dh)
    got = torch.empty(M, 2 * H, dtype=torch.bfloat16, device="cuda")
    amax = torch.zeros(1, dtype=torch.int32, device="cuda")
    ops.gemm(ac, bc, M=M, N=H, K=K, b_mn=True, a_scale=sa, b_scale=sb, epi=ops.EPI_SWIGLU_BWD, out=got, res=gu,
             amax=amax)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int16), want.view(torch.int16))
    assert amax.item() == slot.item()


@pytest.mark.parametrize("acc", [False, True])
def test_gemm_tail_split_matches_single_launch(ops, acc):
    """qtk_gemm's tail split (gemm.cu tail_plan) at the 0.5B gate_up wgrad shape
    (M 9728 x N 896 x K 16384, both operands MN-major, E5M2 x E4M3): 152 pair tiles on
    74 pairs run as a 148-tile head launch + the last M panel split-K 16 ways + the
    deterministic reduce.  Against the single launch (itself checked against the
    reference in test_bench_shapes_gpu.py): <= 1 bf16 ulp everywhere, >= 99.9 % bit-equal
    (only the f32 summation order of the tail rows differs); the SR-accumulate epilogue
    keeps the unsplit GEMM's counters, so the accumulate variant agrees the same way."""
    T, F, d = 16384, 9728, 896
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randint(0, 120, (T, F), dtype=torch.uint8, device="cuda", generator=g)
    b = torch.randint(0, 120, (T, d), dtype=torch.uint8, device="cuda", generator=g)
    sa = torch.tensor([3.0], device="cuda")
    sb = torch.tensor([5.0], device="cuda")
    kw = dict(M=F, N=d, K=T, a_mn=True, b_mn=True, a_fmt=1, a_scale=sa, b_scale=sb)
    acc0 = (torch.randn(F, d, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    if acc:
        kw.update(epi=ops.EPI_BF16_ACC, sr=(7, 11, 123456))
    mh, st = ops.gemm_tail_plan(a, b, split_k=0, **kw)
    assert (mh, st) == (37 * 256, 16), (mh, st)
    assert ops.gemm_tail_plan(a, b, split_k=1, **kw) == (F, 1)
    outs = []
    for sk in (1, 0):
        o = acc0.clone() if acc else None
        outs.append(ops.gemm(a, b, split_k=sk, out=o, **kw).float().cpu().numpy())
    du = _ulp_diff(outs[0], outs[1])
    assert du.max() <= 1, du.max()
    assert (du == 0).mean() >= 0.999, (du == 0).mean()
    assert (du[:mh] == 0).all()  # the head rows are the same launch shape: bit-identical
