"""AdamW, gradient norm and GradAccumulator on device vs the reference on
IDENTICAL gradients (src/optim.cpp:37-110, src/model.cpp:448-464).
AdamW and the SR writes are bit-exact; the f64 norm matches to 1e-12."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = dict(n_layers=2, d_model=128, d_ff=256, n_heads=2, n_kv_heads=1, vocab=256, seq_len=64)


def _session(moments="f32", seed=7):
    from paper_2512_15306_b200 import session as S
    cfg = S.ModelConfig(**SMALL)
    s = S.Session(cfg, plan=S.RunPlan(micro_batch=2, moments=moments), hyper=S.AdamWHyper(lr=1e-3, weight_decay=0.1),
                  seed=seed)
    s.init_params(seed)
    toks = np.random.default_rng(1).integers(0, cfg.vocab, size=2 * (cfg.seq_len + 1), dtype=np.int32)
    s.build_step_context()
    s.zero_grads()
    s.forward(toks, 2)
    s.backward(0)
    return s


def test_adamw_bitexact(ref):
    s = _session()
    before = {n: s.download(n) for n in s.names}
    grads = {n: s.grad(n) for n in s.names}
    scale = 0.37
    s.adamw_step(scale)
    for n in s.names:
        p, m, v = ref.adamw_tensor(n, before[n], np.zeros_like(before[n]), np.zeros_like(before[n]), grads[n],
                                   lr=1e-3, wd=0.1, seed=7, step_count=0, grad_scale=scale)
        np.testing.assert_array_equal(s.download(n), p, err_msg=n)
        gm, gv = s.moments(n)
        np.testing.assert_array_equal(gm, m, err_msg=n)
        np.testing.assert_array_equal(gv, v, err_msg=n)


def test_adamw_second_step_bitexact(ref):
    """bias corrections and SR counters advance with the step (src/optim.cpp:35-36,140-149)."""
    s = _session()
    s.adamw_step(1.0)
    p1 = {n: s.download(n) for n in s.names}
    m1 = {n: s.moments(n) for n in s.names}
    grads = {n: s.grad(n) for n in s.names}
    s.adamw_step(0.5)
    for n in s.names:
        p, m, v = ref.adamw_tensor(n, p1[n], m1[n][0], m1[n][1], grads[n], lr=1e-3, wd=0.1, seed=7, step_count=1,
                                   grad_scale=0.5)
        np.testing.assert_array_equal(s.download(n), p, err_msg=n)


def test_grad_norm_matches_reference(ref):
    s = _session()
    grads = {n: s.grad(n) for n in s.names}
    want = np.sqrt(sum(ref.grad_norm_partials(grads[n]) for n in sorted(grads)))  # std::map name order
    got = s.grad_norm()
    assert abs(got - want) / want < 1e-12, (got, want)


def test_nonfinite_gradient_raises():
    from paper_2512_15306_b200 import session as S
    s = _session()
    with pytest.raises(S.QtError, match="non-finite gradient"):
        s.adamw_step(float("inf"))


@pytest.mark.parametrize("W", [2, 3, 5])
@pytest.mark.parametrize("stochastic", [True, False])
def test_reduce_scatter_sr_matches_reference(ref, W, stochastic):
    """qtk_reduce_scatter_sr == reduce_scatter_oracle (src/comms.cpp:233-254),
    every shard, bit for bit."""
    import ctypes as C
    from paper_2512_15306_b200 import _lib
    from tests.helpers import bf16_grid_round, rng_floats
    n = 3001
    chunks = bf16_grid_round(rng_floats(40 + W, W * W * n, -1, 1)).reshape(W, W, n)
    acc = bf16_grid_round(rng_floats(50 + W, W * n, -0.5, 0.5)).reshape(W, n)
    want = ref.reduce_scatter(chunks, acc, stochastic=stochastic, seed=7, step=5, layer=2)
    dev_chunks = torch.from_numpy(chunks).cuda().to(torch.bfloat16)
    for w in range(W):
        a = torch.from_numpy(acc[w].copy()).cuda()
        srcs = (C.c_void_p * W)(*[dev_chunks[i, w].data_ptr() for i in range(W)])
        rc = _lib.lib().qtk_reduce_scatter_sr(a.data_ptr(), srcs, W, w, n, int(stochastic), 7, 5, 2,
                                              torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        np.testing.assert_array_equal(a.cpu().numpy(), want[w])
