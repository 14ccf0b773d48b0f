"""Per-tensor backward diagnostics vs the reference (dev tool)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import ref
from paper_2512_15306_b200 import session as S

def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = S.ModelConfig(n_layers=L, d_model=128, d_ff=256, n_heads=2, n_kv_heads=1, vocab=256, seq_len=64)
B = 2
rm = ref.RefModel(cfg.as_list(), 1234)
s = S.Session(cfg, plan=S.RunPlan(micro_batch=B), seed=1234)
for n in rm.names: s.upload(n, rm.get(n))
toks = np.random.default_rng(5).integers(0, cfg.vocab, size=B * (cfg.seq_len + 1), dtype=np.int32)
rm.fwd_bwd(toks, B)
s.build_step_context(); s.zero_grads(); s.forward(toks, B); s.backward(0)
for n in rm.names:
    g = rm.grad(n)
    want = ref.grad_accumulate(n, np.zeros_like(g), g, seed=1234, micro_step=0)
    got = s.grad(n)
    print(f"{n:24s} rel {rel(got, want):.3e}  exact {(got == want).mean():.4f}  |ref| {np.linalg.norm(want):.3e} |got| {np.linalg.norm(got):.3e}")
# lm_head detail
n = "lm_head"; g = rm.grad(n)
want = ref.grad_accumulate(n, np.zeros_like(g), g, seed=1234, micro_step=0).reshape(cfg.vocab, -1)
got = s.grad(n).reshape(cfg.vocab, -1); g = g.reshape(cfg.vocab, -1)
tg = set(toks.reshape(B, -1)[:, 1:].ravel().tolist())
rowerr = np.linalg.norm(got - want, axis=1) / (np.linalg.norm(want, axis=1) + 1e-30)
ist = np.array([v in tg for v in range(cfg.vocab)])
print("target rows err", rowerr[ist].mean(), "non-target rows err", rowerr[~ist].mean())
print("raw vs ours rel", rel(got, g), "raw vs want rel", rel(want, g))
worst = np.argsort(-rowerr)[:5]
for v in worst: print(v, v in tg, rowerr[v], got[v, :4], want[v, :4], g[v, :4])
nf_ref = ref.rmsnorm_residual_fused(None, rm.saved(0, "r_final").reshape(B * cfg.seq_len, -1), rm.get("final_g"))[1]
nf = s.saved(0, "normed_final")
print("normed_final rel", rel(nf, nf_ref.ravel()), "exact", (nf == nf_ref.ravel()).mean())
lg = s.saved(0, "logits").reshape(B * cfg.seq_len, -1)
lref = ref.matmul_f32(nf_ref.reshape(B * cfg.seq_len, -1), rm.get("lm_head").reshape(cfg.vocab, -1), round_bf16=False)
print("logits rel", rel(lg, lref))
dl = s.saved(0, "dlogits") + s.saved(0, "dlogits_lo")
N = B * cfg.seq_len
tg = toks.reshape(B, -1)[:, 1:].ravel()
mx = lref.max(1, keepdims=True); e = np.exp(lref - mx); p = e / e.sum(1, keepdims=True); p[np.arange(N), tg] -= 1; p /= N
print("dlogits rel", rel(dl, p.ravel()))
dh = s.saved(0, "d_hidden"); print("d_hidden rel", rel(dh, rm.saved(0, "d_hidden")))
dw = p.T.astype(np.float64) @ nf_ref.reshape(N, -1).astype(np.float64)
print("dw(np from p, nf) vs raw ref", rel(dw.ravel(), rm.grad("lm_head")))
