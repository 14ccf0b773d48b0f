"""Tiny-config (BASELINE configs[0]) one-step gradient errors vs the reference,
to compare with SURVEY.md Appendix P6's oracle order-noise floor."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import ref
from paper_2512_15306_b200 import session as S
def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
cfg = S.PRESETS["tiny"]; B = 4
e5 = True
rm = ref.RefModel(cfg.as_list(), 1234, grad_e5m2=e5)
s = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2" if e5 else "e4m3"), S.RunPlan(micro_batch=B), seed=1234)
for n in rm.names: s.upload(n, rm.get(n))
toks = np.random.default_rng(0).integers(0, cfg.vocab, size=B * (cfg.seq_len + 1), dtype=np.int32)
lw = rm.fwd_bwd(toks, B)
s.build_step_context(); s.zero_grads(); lg = s.forward(toks, B); s.backward(0)
print("loss", lg, lw, (lg - lw) / lw)
for n in rm.names:
    g = rm.grad(n)
    want = ref.grad_accumulate(n, np.zeros_like(g), g, seed=1234, micro_step=0)
    print(f"{n:24s} rel {rel(s.grad(n), want):.3e}")
