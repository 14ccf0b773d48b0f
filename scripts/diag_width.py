"""Per-site forward comparison against the reference at a real width (1 layer, few
tokens): which activation first departs from the reference by more than bf16 ulps."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import ref
from paper_2512_15306_b200 import session as S
preset = sys.argv[1] if len(sys.argv) > 1 else "llama-7b"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16
p = S.PRESETS[preset]
cfg = S.ModelConfig(n_layers=1, d_model=p.d_model, d_ff=p.d_ff, n_heads=p.n_heads, n_kv_heads=p.n_kv_heads,
                    vocab=p.vocab, seq_len=T)
rm = ref.RefModel(cfg.as_list(), 1234, grad_e5m2=True)
sess = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), S.RunPlan(micro_batch=1), seed=1234)
for n in rm.names:
    sess.upload(n, rm.get(n))
toks = np.random.default_rng(31).integers(0, cfg.vocab, size=T + 1, dtype=np.int32)
lw = rm.fwd_bwd(toks, 1)
sess.build_step_context()
sess.zero_grads()
lg = sess.forward(toks, 1)
sess.backward(0)
print(f"{preset} T={T}: loss ref {lw:.6f} ours {lg:.6f} rel {abs(lg - lw) / lw:.2e}")


def ulp(a, b):
    ai = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64) >> 16
    bi = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64) >> 16
    return np.abs(ai - bi)


for site in ("r_in", "qkv", "att", "r_mid", "gate_up"):
    w, g = rm.saved(0, site), sess.saved(0, site)
    if w is None or g is None:
        continue
    g = np.asarray(g, np.float32).ravel()[: w.size]
    u = ulp(g, w)
    print(f"  {site:8s} rel {np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-30):.2e} exact {(u == 0).mean():.4f} "
          f"<=1 {(u <= 1).mean():.4f} max {u.max()}")
for n in rm.names:
    w = rm.grad(n)
    g = sess.grad(n)
    acc = ref.grad_accumulate(n, np.zeros_like(w), w, seed=1234, micro_step=0)
    print(f"  grad {n:20s} rel(vs SR'd ref) {np.linalg.norm(g - acc) / max(np.linalg.norm(acc), 1e-30):.3e}")
