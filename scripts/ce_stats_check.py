import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2512_15306_b200 import ops
for (N, d, V) in [(256, 128, 1000), (300, 256, 4100), (1024, 896, 151936)]:
    g = torch.Generator(device="cpu").manual_seed(3)
    h = (torch.randn(N, d, generator=g) * 0.5).to(torch.bfloat16).cuda()
    w = (torch.randn(V, d, generator=g) * 0.5).to(torch.bfloat16).cuda()
    t = torch.randint(0, V, (N,), generator=g, dtype=torch.int32).cuda()
    stats = torch.empty(N, (V + 127) // 128, 2, dtype=torch.float32, device="cuda")
    tl = torch.empty(N, dtype=torch.float32, device="cuda")
    logits = ops.gemm(h, w, M=N, N=V, K=d, epi=ops.EPI_F32, ce=(t, stats, tl))
    l2, hi2, lo2 = ops.ce_softmax(logits, t, 1.0 / N)
    l1, hi1, lo1 = ops.ce_softmax_stats(logits, t, stats, tl, 1.0 / N)
    torch.cuda.synchronize()
    f1 = hi1.float() + lo1.float(); f2 = hi2.float() + lo2.float()
    rel = ((f1 - f2).abs() / f2.abs().clamp_min(1e-30)).max().item()
    print(N, d, V, "loss rel", ((l1 - l2).abs() / l2.abs()).max().item(), "dl max rel", rel,
          "hi same", (hi1.view(torch.int16) == hi2.view(torch.int16)).float().mean().item(),
          "tl ok", torch.equal(tl, logits[torch.arange(N), t.long()]), "logit range", logits.abs().max().item())
