import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from oracle import ref
from paper_2512_15306_b200 import ops
from tests.helpers import rng_floats
def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
N, d, V = 128, 128, 256
h = rng_floats(1, N * d, -1, 1).reshape(N, d); w = rng_floats(2, V * d, -0.2, 0.2).reshape(V, d)
t = np.random.default_rng(3).integers(0, V, N).astype(np.int32)
loss, dh, dw = ref.cross_entropy(h, w, t)
H = torch.from_numpy(h).cuda().bfloat16(); W = torch.from_numpy(w).cuda().bfloat16(); Tt = torch.from_numpy(t).cuda()
logits = ops.gemm(H, W, M=N, N=V, K=d, epi=ops.EPI_F32)
ref_logits = ref.matmul_f32(h, w, round_bf16=False)
print("logits rel", rel(logits.cpu().numpy(), ref_logits))
lr, hi, lo = ops.ce_softmax(logits, Tt, 1.0 / N)
print("loss", lr.mean().item(), loss)
dl = hi.float() + lo.float()
# reference dlogits
mx = ref_logits.max(1, keepdims=True); e = np.exp(ref_logits - mx); p = e / e.sum(1, keepdims=True); p[np.arange(N), t] -= 1; p /= N
print("dlogits rel", rel(dl.cpu().numpy(), p), "hi-only rel", rel(hi.float().cpu().numpy(), p))
dh_g = ops.gemm(hi, W, M=N, N=d, K=V, b_mn=True, epi=ops.EPI_BF16, a2=lo)
print("d_hidden rel", rel(dh_g.float().cpu().numpy(), dh), "exact", (dh_g.float().cpu().numpy() == dh).mean())
dh_g1 = ops.gemm(hi, W, M=N, N=d, K=V, b_mn=True, epi=ops.EPI_BF16)
print("d_hidden hi-only rel", rel(dh_g1.float().cpu().numpy(), dh))
dw_g = ops.gemm(hi, H, M=V, N=d, K=N, a_mn=True, b_mn=True, epi=ops.EPI_F32, a2=lo)
print("d_lm_w rel", rel(dw_g.cpu().numpy(), dw))
dw_g1 = ops.gemm(hi, H, M=V, N=d, K=N, a_mn=True, b_mn=True, epi=ops.EPI_F32)
print("d_lm_w hi-only rel", rel(dw_g1.cpu().numpy(), dw))
dw_t = (dl.T @ H.float()).cpu().numpy()
print("d_lm_w torch f32 on (hi+lo) rel", rel(dw_t, dw))
