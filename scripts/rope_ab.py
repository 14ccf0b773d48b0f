"""RoPE kernel A/B (qtk_rope_set_heads 0 / 1) at the 0.5B and 7B shapes, forward and
backward-with-absmax; CUDA events, 20 calls, median of 5."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2512_15306_b200 import _lib
L = _lib.lib()
for name, (rows, T, H, Hkv, hd) in (("0.5b", (16384, 1024, 14, 2, 64)), ("7b", (8192, 1024, 32, 32, 128))):
    q = (H + 2 * Hkv) * hd
    x = torch.randn(rows, q, device="cuda").to(torch.bfloat16)
    tab = torch.randn(T, hd // 2, 2, device="cuda")
    am = torch.zeros(1, dtype=torch.int32, device="cuda")
    for bwd in (0, 1):
        res = []
        for mode in (0, 1):
            L.qtk_rope_set_heads(mode)
            f = lambda: L.qtk_rope(x.data_ptr(), rows, T, H + Hkv, hd, q, tab.data_ptr(), bwd,
                                   am.data_ptr() if bwd else None, torch.cuda.current_stream().cuda_stream)
            f()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    f()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 20 * 1e3)
            res.append(sorted(ts)[2])
        print(f"{name} {'bwd' if bwd else 'fwd'}: per-item {res[0]:.1f} us, head-looped {res[1]:.1f} us", flush=True)
L.qtk_rope_set_heads(1)
