"""Thin torch-facing wrappers over the stateless C-ABI kernels (qtk_*).

torch is used only for device allocation and the current stream; every
computation runs in the native library.  Tensors must already be on the GPU.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib

E4M3, E5M2 = 0, 1
EPI_BF16, EPI_F32, EPI_BF16_RES, EPI_BF16_ACC, EPI_F32_ACC, EPI_SWIGLU_BWD = 0, 1, 2, 3, 4, 5


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _s() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("qtrain-b200 kernels take CUDA tensors (no CPU fallback)")


def absmax(x: torch.Tensor, slot: torch.Tensor | None = None) -> torch.Tensor:
    """Returns a 1-element int32 tensor holding the f32 bit pattern of max|x|."""
    _need_cuda(x)
    if slot is None:
        slot = torch.zeros(1, dtype=torch.int32, device=x.device)
    if x.dtype == torch.bfloat16:
        rc = _lib.lib().qtk_absmax_bf16(_p(x), x.numel(), _p(slot), _s())
    elif x.dtype == torch.float32:
        rc = _lib.lib().qtk_absmax_f32(_p(x), x.numel(), _p(slot), _s())
    else:
        raise TypeError(x.dtype)
    _lib.check(rc, "qtk_absmax")
    return slot


def amax_value(slot: torch.Tensor) -> float:
    return slot.view(torch.float32).item()


def quantize(x: torch.Tensor, kind: int, slot: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    _need_cuda(x)
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    scale = torch.empty(1, dtype=torch.float32, device=x.device)
    rc = _lib.lib().qtk_quantize_bf16(_p(x), x.numel(), kind, _p(slot), _p(codes), _p(scale), _s())
    _lib.check(rc, "qtk_quantize_bf16")
    return codes, scale


def quantize_transpose(x: torch.Tensor, kind: int, slot: torch.Tensor, with_rowmajor: bool = False):
    _need_cuda(x)
    rows, cols = x.shape
    ct = torch.empty((cols, rows), dtype=torch.uint8, device=x.device)
    crm = torch.empty((rows, cols), dtype=torch.uint8, device=x.device) if with_rowmajor else None
    scale = torch.empty(1, dtype=torch.float32, device=x.device)
    rc = _lib.lib().qtk_quantize_transpose_bf16(_p(x), rows, cols, kind, _p(slot), _p(ct), _p(crm), _p(scale), _s())
    _lib.check(rc, "qtk_quantize_transpose_bf16")
    return ct, crm, scale


def gemm(a: torch.Tensor, b: torch.Tensor, *, M: int, N: int, K: int, a_mn: bool = False, b_mn: bool = False,
         a_fmt: int = E4M3, b_fmt: int = E4M3, a_scale: torch.Tensor | None = None,
         b_scale: torch.Tensor | None = None, epi: int = EPI_BF16, out: torch.Tensor | None = None,
         res: torch.Tensor | None = None, sr: tuple[int, int, int] = (0, 0, 0), bn: int = 0,
         a2: torch.Tensor | None = None, split_k: int = 1, amax: torch.Tensor | None = None,
         ce: tuple | None = None) -> torch.Tensor:
    """D[m,n] = sum_k A[m,k] B[n,k].  A stored [M][K] (a_mn=False) or [K][M]
    (a_mn=True); likewise B.  uint8 operands are FP8 codes, bf16 operands BF16."""
    g, out, ws = _gemm_desc(a, b, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, a_fmt=a_fmt, b_fmt=b_fmt, a_scale=a_scale,
                            b_scale=b_scale, epi=epi, out=out, res=res, sr=sr, bn=bn, a2=a2, split_k=split_k,
                            amax=amax, ce=ce)
    _lib.check(_lib.lib().qtk_gemm(C.byref(g), _s()), "qtk_gemm")
    return out


def gemm_plan(a: torch.Tensor, b: torch.Tensor, **kw) -> dict:
    """The instantiation qtk_gemm would launch for the same arguments as gemm()
    (qtk_gemm_plan shares qtk_gemm's decision): cta_group, BN, split-K factor,
    grid and output tiles per CTA of the persistent loop."""
    g, _, _ = _gemm_desc(a, b, **kw)
    o = [C.c_int() for _ in range(5)]
    _lib.check(_lib.lib().qtk_gemm_plan(C.byref(g), *[C.byref(x) for x in o]), "qtk_gemm_plan")
    return dict(zip(("cg", "bn", "splits", "grid", "tiles_per_cta"), (x.value for x in o)))


def gemm_tail_plan(a: torch.Tensor, b: torch.Tensor, **kw) -> tuple[int, int]:
    """(head rows, tail split-K factor) when qtk_gemm runs the same arguments as a
    tail split (head launch + split-K tail), else (M, 1)."""
    g, _, _ = _gemm_desc(a, b, **kw)
    mh, st = C.c_int64(), C.c_int()
    on = _lib.lib().qtk_gemm_tail_plan(C.byref(g), C.byref(mh), C.byref(st))
    return (mh.value, st.value) if on else (kw["M"], 1)


def _gemm_desc(a, b, *, M, N, K, a_mn=False, b_mn=False, a_fmt=E4M3, b_fmt=E4M3, a_scale=None, b_scale=None,
               epi=EPI_BF16, out=None, res=None, sr=(0, 0, 0), bn=0, a2=None, split_k=1, amax=None, ce=None):
    _need_cuda(a, b)
    kind = 0 if a.dtype == torch.uint8 else 1
    if out is None:
        dt = torch.float32 if epi == EPI_F32 else torch.bfloat16
        out = torch.empty((M, N), dtype=dt, device=a.device)
    g = _lib.QtkGemm()
    g.kind, g.a_fmt, g.b_fmt, g.a_mn, g.b_mn = kind, a_fmt, b_fmt, int(a_mn), int(b_mn)
    g.M, g.N, g.K = M, N, K
    g.a, g.lda = _p(a), a.stride(0)
    g.b, g.ldb = _p(b), b.stride(0)
    g.a_scale, g.b_scale = _p(a_scale), _p(b_scale)
    g.epi, g.out, g.ldo = epi, _p(out), out.stride(0)
    g.res, g.ldr = _p(res), (res.stride(0) if res is not None else 0)
    g.sr_seed, g.sr_stream, g.sr_base = sr
    g.bn = bn
    g.a2 = _p(a2)
    ws = None
    if split_k != 1:
        nbytes = _lib.lib().qtk_gemm_splitk_ws_bytes(M, N, K, kind)
        if split_k > 1:
            nbytes = split_k * M * N * 4
        if nbytes > 0:
            ws = torch.empty(nbytes // 4, dtype=torch.float32, device=a.device)
            g.ws, g.ws_bytes = _p(ws), nbytes
    g.split_k = split_k
    g.amax = _p(amax)
    if ce is not None:  # (targets, stats, tgt_logit): softmax statistics in the logits epilogue
        g.ce_targets, g.ce_stats, g.ce_tgt_logit = _p(ce[0]), _p(ce[1]), _p(ce[2])
    return g, out, ws


def ce_softmax(logits: torch.Tensor, targets: torch.Tensor, inv_n: float, with_grads: bool = True):
    """Per-row CE loss and dlogits (bf16 hi, bf16 lo) from f32 logits."""
    _need_cuda(logits, targets)
    rows, V = logits.shape
    loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
    hi = torch.empty((rows, V), dtype=torch.bfloat16, device=logits.device) if with_grads else None
    lo = torch.empty((rows, V), dtype=torch.bfloat16, device=logits.device) if with_grads else None
    rc = _lib.lib().qtk_ce_softmax(_p(logits), logits.stride(0), rows, V, _p(targets), inv_n, _p(hi), _p(lo), V,
                                   _p(loss), _s())
    _lib.check(rc, "qtk_ce_softmax")
    return loss, hi, lo


def ce_softmax_stats(logits, targets, stats, tgt_logit, inv_n: float):
    """ce_softmax from the statistics the logits GEMM produced (single pass over the logits)."""
    rows, V = logits.shape
    loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
    hi = torch.empty((rows, V), dtype=torch.bfloat16, device=logits.device)
    lo = torch.empty((rows, V), dtype=torch.bfloat16, device=logits.device)
    rc = _lib.lib().qtk_ce_softmax_stats(_p(logits), logits.stride(0), rows, V, _p(targets), _p(stats),
                                         _p(tgt_logit), inv_n, _p(hi), _p(lo), V, _p(loss), _s())
    _lib.check(rc, "qtk_ce_softmax_stats")
    return loss, hi, lo


def ce_softmax_stats_tx(logits, targets, stats, tgt_logit, inv_n: float):
    """Target-exact CE softmax: per-row loss, bf16 dlogits with the target entry
    zeroed, and the f32 target term dl_t = (p_t - 1) / N."""
    rows, V = logits.shape
    loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
    dl = torch.empty((rows, V), dtype=torch.bfloat16, device=logits.device)
    dlt = torch.empty(rows, dtype=torch.float32, device=logits.device)
    rc = _lib.lib().qtk_ce_softmax_stats_tx(_p(logits), logits.stride(0), rows, V, _p(targets), _p(stats),
                                            _p(tgt_logit), inv_n, _p(dl), V, _p(loss), _p(dlt), _s())
    _lib.check(rc, "qtk_ce_softmax_stats_tx")
    return loss, dl, dlt


def embed_sort(ids: torch.Tensor, V: int):
    """Stable sort of positions by id (qtk_embed_sort): sorted_pos, seg_tok,
    seg_off, nseg (device tensors)."""
    n = ids.numel()
    L = _lib.lib()
    nb = L.qtk_embed_sort_scratch_bytes(n, V)
    scratch = torch.empty(max(nb, 1), dtype=torch.uint8, device=ids.device)
    sp = torch.empty(n, dtype=torch.int32, device=ids.device)
    st = torch.empty(n, dtype=torch.int32, device=ids.device)
    so = torch.empty(n + 1, dtype=torch.int32, device=ids.device)
    ns = torch.zeros(4, dtype=torch.int32, device=ids.device)
    _lib.check(L.qtk_embed_sort(_p(ids), n, V, _p(scratch), nb, _p(sp), _p(st), _p(so), _p(ns), _s()),
               "qtk_embed_sort")
    return sp, st, so, ns


def lm_splits(V: int) -> int:
    """The session's split-K factor for the LM-head dgrad (K = V)."""
    return int(min(8, max(1, -(-V // 16384))))


def lm_dgrad_tx(dl, dl_t, targets, lm_w):
    """d_hidden of the target-exact CE backward, as the session runs it: split-K
    f32 GEMM of the bf16 dlogits, then + dl_t * lm_w[target], rounded to bf16."""
    M, V = dl.shape
    d = lm_w.shape[1]
    acc = gemm(dl, lm_w, M=M, N=d, K=V, b_mn=True, epi=EPI_F32, split_k=lm_splits(V))
    out = torch.empty((M, d), dtype=torch.bfloat16, device=dl.device)
    _lib.check(_lib.lib().qtk_lm_dgrad_finish(_p(acc), M, d, _p(dl_t), _p(targets), _p(lm_w), _p(out), _s()),
               "qtk_lm_dgrad_finish")
    return out


def lm_wgrad_tx(dl, dl_t, targets, hidden):
    """f32 d_lm_w of the target-exact CE backward: GEMM of the bf16 dlogits
    (target entries zero) + the exact target terms in ascending token order."""
    M, V = dl.shape
    d = hidden.shape[1]
    acc = gemm(dl, hidden, M=V, N=d, K=M, a_mn=True, b_mn=True, epi=EPI_F32)
    sp, st, so, ns = embed_sort(targets, V)
    _lib.check(_lib.lib().qtk_lm_wgrad_targets(_p(acc), d, _p(sp), _p(st), _p(so), _p(ns), M, _p(dl_t), _p(hidden),
                                               _s()), "qtk_lm_wgrad_targets")
    return acc


def rmsnorm_fwd(x, res, gamma, eps=1e-6, with_absmax=True):
    rows, d = res.shape
    nr = torch.empty_like(res) if x is not None else None
    normed = torch.empty_like(res)
    slot = torch.zeros(1, dtype=torch.int32, device=res.device) if with_absmax else None
    inv = torch.empty(rows, dtype=torch.float32, device=res.device)
    rc = _lib.lib().qtk_rmsnorm_fwd(_p(x), _p(res), _p(gamma), rows, d, eps, _p(nr), _p(normed), _p(inv), _p(slot),
                                    _s())
    _lib.check(rc, "qtk_rmsnorm_fwd")
    return nr, normed, slot


def rmsnorm_bwd(nr, gamma, dy, d_extra=None, eps=1e-6):
    rows, d = nr.shape
    nblk = _lib.lib().qtk_rmsnorm_bwd_partials(rows, d)
    part = torch.empty((nblk, d), dtype=torch.float32, device=nr.device)
    dg = torch.empty(d, dtype=torch.float32, device=nr.device)
    din = torch.empty_like(nr)
    slot = torch.zeros(1, dtype=torch.int32, device=nr.device)
    rc = _lib.lib().qtk_rmsnorm_bwd(_p(nr), _p(gamma), rows, d, eps, _p(dy), _p(d_extra), _p(din), _p(part), _p(dg),
                                    _p(slot), _s())
    _lib.check(rc, "qtk_rmsnorm_bwd")
    return din, dg, slot


def swiglu_fwd(gu):
    rows, two_h = gu.shape
    h = torch.empty((rows, two_h // 2), dtype=torch.bfloat16, device=gu.device)
    slot = torch.zeros(1, dtype=torch.int32, device=gu.device)
    _lib.check(_lib.lib().qtk_swiglu_fwd(_p(gu), rows, two_h // 2, _p(h), _p(slot), _s()), "qtk_swiglu_fwd")
    return h, slot


def swiglu_bwd(gu, dh):
    rows, two_h = gu.shape
    out = torch.empty_like(gu)
    slot = torch.zeros(1, dtype=torch.int32, device=gu.device)
    _lib.check(_lib.lib().qtk_swiglu_bwd(_p(gu), _p(dh), rows, two_h // 2, _p(out), _p(slot), _s()), "qtk_swiglu_bwd")
    return out, slot


def attn_fwd(qkv, B, T, H, Hkv, hd):
    rows, qkv_dim = qkv.shape
    d = H * hd
    out = torch.empty((rows, d), dtype=torch.bfloat16, device=qkv.device)
    out32 = torch.empty((rows, d), dtype=torch.float32, device=qkv.device)
    lse = torch.empty((B, H, T), dtype=torch.float32, device=qkv.device)
    slot = torch.zeros(1, dtype=torch.int32, device=qkv.device)
    rc = _lib.lib().qtk_attn_fwd(_p(qkv), B, T, H, Hkv, hd, qkv_dim, _p(out), d, _p(out32), _p(lse), _p(slot), _s())
    _lib.check(rc, "qtk_attn_fwd")
    return out, out32, lse, slot


def attn_bwd(qkv, out32, dout, lse, B, T, H, Hkv, hd):
    rows, qkv_dim = qkv.shape
    d = H * hd
    Dv = torch.empty((B, H, T), dtype=torch.float32, device=qkv.device)
    dqkv = torch.zeros_like(qkv)
    wsb = _lib.lib().qtk_attn_bwd_ws_bytes(B, T, H, Hkv, hd)
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=qkv.device)
    rc = _lib.lib().qtk_attn_bwd(_p(qkv), _p(out32), _p(dout), d, _p(lse), _p(Dv), B, T, H, Hkv, hd, qkv_dim,
                                 _p(dqkv), _p(ws), _s())
    _lib.check(rc, "qtk_attn_bwd")
    return dqkv
