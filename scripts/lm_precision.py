"""LM-head backward precision diagnostic (GPU): d_hidden = dlogits . lm_w with
realistic CE dlogits (p - onehot)/N at V = 151936, compared with the exact
(f64) product of the same operands rounded to bf16, for the reference's
sequential f32 matmul and for the device split-A GEMM at several split-K
factors, plus the bf16-only (no lo part) variant."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2512_15306_b200 import ops
from oracle import ref
from tests.helpers import bf16_grid_round

M, d, V = int(sys.argv[1]) if len(sys.argv) > 1 else 512, 896, 151936
torch.manual_seed(0)
h = torch.randn(M, d, device="cuda").to(torch.bfloat16)
w = (torch.randn(V, d, device="cuda") * d ** -0.5).to(torch.bfloat16)
t = torch.randint(0, V, (M,), device="cuda")
logits = h.float() @ w.float().T
p = torch.softmax(logits, dim=1)
p[torch.arange(M), t] -= 1.0
dl = p / M
hi = dl.to(torch.bfloat16)
lo = (dl - hi.float()).to(torch.bfloat16)
rows = np.arange(0, M, max(1, M // 16))
ri = torch.from_numpy(rows).cuda()
a = (hi[ri].double() + lo[ri].double())
exact = (a @ w.double()).cpu().numpy()
ex_b = bf16_grid_round(exact.astype(np.float32))


def ulp(x, y):
    xi = np.ascontiguousarray(x, np.float32).view(np.int32).astype(np.int64) >> 16
    yi = np.ascontiguousarray(y, np.float32).view(np.int32).astype(np.int64) >> 16
    return np.abs(xi - yi)


def report(name, got):
    u = ulp(got, ex_b)
    rel = np.linalg.norm(got - exact) / np.linalg.norm(exact)
    print(f"{name:28s} exact {np.mean(u == 0):.5f}  <=1ulp {np.mean(u <= 1):.5f}  max {u.max()}  rel {rel:.2e}")


af = a.float().cpu().numpy()
wf = w.float().cpu().numpy()
report("reference matmul_f32", ref.matmul_f32(af, wf.T.copy(), round_bf16=True))
for sk in (1, 2, 4, 8):
    out = ops.gemm(hi, w, M=M, N=d, K=V, b_mn=True, epi=ops.EPI_BF16, a2=lo, split_k=sk)
    report(f"device split-A split_k={sk}", out[ri].float().cpu().numpy())
out = ops.gemm(hi, w, M=M, N=d, K=V, b_mn=True, epi=ops.EPI_BF16)
report("device bf16-only (no lo)", out[ri].float().cpu().numpy())
# the target column excluded from the GEMM operand (its term would be added in f32 by the epilogue)
hi0, lo0 = hi.clone(), lo.clone()
hi0[torch.arange(M), t] = 0
lo0[torch.arange(M), t] = 0
a0 = (hi0[ri].double() + lo0[ri].double())
ex0 = (a0 @ w.double()).cpu().numpy()
for sk in (1, 4):
    o = ops.gemm(hi0, w, M=M, N=d, K=V, b_mn=True, epi=ops.EPI_F32, a2=lo0, split_k=sk)[ri].double().cpu().numpy()
    # add the target term exactly as the epilogue would: f32 fma of dl_t * w_t
    dl_t = dl[ri, t[ri]].double().cpu().numpy()[:, None]
    wt = w[t[ri]].double().cpu().numpy()
    tot = (o + dl_t * wt).astype(np.float32)
    exact_full = ex0 + dl_t * wt
    u = ulp(bf16_grid_round(tot), bf16_grid_round(exact_full.astype(np.float32)))
    e = o - ex0
    print(f"target excluded split_k={sk}: exact {np.mean(u == 0):.5f} max {u.max()} gemm-part rms err/rms {np.sqrt((e**2).mean()/(ex0**2).mean()):.2e}")
# truncation check on f32 output: device split_k=1 with f32 epilogue vs exact
out32 = ops.gemm(hi, w, M=M, N=d, K=V, b_mn=True, epi=ops.EPI_F32, a2=lo)
e = out32[ri].double().cpu().numpy() - exact
print("f32 out: mean signed err / mean |exact|", e.mean() / np.abs(exact).mean(), " rms err/rms", np.sqrt((e ** 2).mean() / (exact ** 2).mean()))
e2 = ref.matmul_f32(af, wf.T.copy(), round_bf16=False) - exact
print("ref f32:  mean signed err / mean |exact|", e2.mean() / np.abs(exact).mean(), " rms err/rms", np.sqrt((e2 ** 2).mean() / (exact ** 2).mean()))

# ---- wgrad: d_lm_w = dlogits^T . x (K = tokens), f32 output (EPI_F32), sampled vocab rows
x = torch.randn(M, d, device="cuda").to(torch.bfloat16)
tv = t.cpu().numpy()
vrows = np.unique(np.concatenate([tv[:8], np.random.default_rng(1).choice(V, 8, replace=False)]))
vi = torch.from_numpy(vrows).cuda()
aw = (hi[:, vi].double() + lo[:, vi].double()).T  # (rows, M)
exw = (aw @ x.double()).cpu().numpy()
print("wgrad (f32 out), vocab rows incl. targets:")
for sk in (1, 2, 4):
    o = ops.gemm(hi, x, M=V, N=d, K=M, a_mn=True, b_mn=True, epi=ops.EPI_F32, a2=lo, split_k=sk)
    e = o[vi].double().cpu().numpy() - exw
    print(f"  device split_k={sk}: rms err/rms {np.sqrt((e ** 2).mean() / (exw ** 2).mean()):.2e}  max |err|/rms {np.abs(e).max() / np.sqrt((exw ** 2).mean()):.2e}")
e2 = ref.matmul_f32(aw.float().cpu().numpy(), x.float().cpu().numpy().T.copy(), round_bf16=False) - exw
print(f"  reference         : rms err/rms {np.sqrt((e2 ** 2).mean() / (exw ** 2).mean()):.2e}  max |err|/rms {np.abs(e2).max() / np.sqrt((exw ** 2).mean()):.2e}")
