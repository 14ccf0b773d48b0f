"""One small FP8 training step on cuda:0 through the native library, checked
against the oracle (used by __graft_entry__.smoke())."""
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
    from oracle import ref as R  # checker only
    rm = R.RefModel(cfg.as_list(), seed, grad_e5m2=True)
    for n in rm.names:
        sess.upload(n, rm.get(n))
    lw, nw = rm.train_step(toks, B, step=0)
    lg, ng = sess.train_step(toks, B, step=0)
    assert abs(lg - lw) / lw < 1e-3, (lg, lw)
    worst = 0.0
    for n in rm.names:
        a, b = sess.download(n).astype(np.float64), rm.get(n).astype(np.float64)
        worst = max(worst, np.linalg.norm(a - b) / np.linalg.norm(b))
    assert worst < 4e-3, worst
    print(f"smoke ok: loss {lg:.6f} vs oracle {lw:.6f}; grad norm {ng:.5f} vs {nw:.5f}; "
          f"max param rel err {worst:.2e}")
