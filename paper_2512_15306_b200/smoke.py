"""One small FP8 training step on cuda:0 through the native library, checked
against the oracle (used by __graft_entry__.smoke()).  The checker is the
unmodified reference (oracle/_ref) when it was built, else the C restatement
(oracle/_build) on the step's first, teacher-forced ops."""
from __future__ import annotations

import numpy as np


def run() -> None:
    import torch

    from . import session as S
    assert torch.cuda.is_available(), "smoke needs cuda:0"
    torch.cuda.set_device(0)
    cfg = S.ModelConfig(n_layers=2, d_model=128, d_ff=256, n_heads=2, n_kv_heads=1, vocab=256, seq_len=64)
    B, seed = 2, 1234
    toks = np.random.default_rng(0).integers(0, cfg.vocab, size=B * (cfg.seq_len + 1), dtype=np.int32)
    sess = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), S.RunPlan(micro_batch=B), seed=seed)
    from oracle import port, ref  # checkers only
    if ref.available():
        rm = ref.RefModel(cfg.as_list(), seed, grad_e5m2=True)
        for n in rm.names:
            sess.upload(n, rm.get(n))
        lw, nw = rm.train_step(toks, B, step=0)
        lg, ng = sess.train_step(toks, B, step=0)
        assert abs(lg - lw) / lw < 1e-3, (lg, lw)
        worst = max(np.linalg.norm(sess.download(n).astype(np.float64) - rm.get(n)) / np.linalg.norm(rm.get(n))
                    for n in rm.names)
        assert worst < 1e-2, worst
        print(f"smoke ok: loss {lg:.6f} vs reference {lw:.6f}; grad norm {ng:.5f} vs {nw:.5f}; "
              f"max param rel err {worst:.2e}")
        return
    sess.init_params(seed)
    std = float(np.float32(1.0) / np.sqrt(np.float32(cfg.d_model)))
    for n in ("embed", "layers.0.w_qkv"):
        assert np.array_equal(sess.download(n), port.init_normal(sess.numel[sess.names.index(n)], std, seed, n))
    sess.build_step_context()
    loss = sess.forward(toks, B)
    d = cfg.d_model
    emb = sess.download("embed").reshape(cfg.vocab, d)
    r0 = emb[toks.reshape(B, -1)[:, :-1].ravel()]
    _, n1, am = port.rmsnorm_residual_fused(None, r0, sess.download("layers.0.ln1_g"))
    codes, _ = port.quantize_with_absmax(n1, 0, am)
    assert np.array_equal(sess.saved(0, "n1c"), codes.ravel())
    assert sess.forward_stats()[0, 0] == am
    sess.backward(0)
    print(f"smoke ok (C-restatement checker): loss {loss:.5f}, layer-0 RMSNorm + E4M3 codes bit-exact")
