"""Sensitivity of the reference itself: flip ONE weight element by one bf16
ulp and measure how far the reference's own gradients move.  FP8 per-tensor
quantization turns tiny upstream differences into discrete code flips, so
this is the natural scale for end-to-end gradient comparisons."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import ref
def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
which = sys.argv[1] if len(sys.argv) > 1 else "small"
if which == "small":
    cfg, B, e5 = [2, 128, 256, 2, 1, 256, 64], 2, False
else:
    cfg, B, e5 = [2, 256, 1536, 4, 4, 512, 256], 4, True
toks = np.random.default_rng(0).integers(0, cfg[5], size=B * (cfg[6] + 1), dtype=np.int32)
a = ref.RefModel(cfg, 1234, grad_e5m2=e5)
la = a.fwd_bwd(toks, B)
ga = {n: a.grad(n) for n in a.names}
b = ref.RefModel(cfg, 1234, grad_e5m2=e5)
w = b.get("layers.0.w_qkv").copy(); i = int(np.argmax(np.abs(w) < 0.5 * np.abs(w).max()))
w[i] = ref.bf16_round(w[i] * 1.125)  # one E4M3 step on one weight element: a single code flip
b.set("layers.0.w_qkv", w)
lb = b.fwd_bwd(toks, B)
print("loss", la, lb, (lb - la) / la)
for n in a.names:
    print(f"{n:24s} {rel(b.grad(n), ga[n]):.3e}")
