"""Tile-configuration sweep of the step's FP8 GEMMs (0.5B and Llama-7B shapes, the
step's epilogues): for each shape every legal (cta_group, BN) the launcher accepts,
device time per call, against the configuration qtk_gemm picks by itself.
Run as: python scripts/gemm_sweep.py  (spawns one process per forced cta_group)."""
import json
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
EPI_BF16, EPI_RES, EPI_ACC = 0, 2, 3


def shapes():
    out = []
    for tag, M, d, q, F in (("0.5b", 16384, 896, 1152, 9728), ("7b", 8192, 4096, 12288, 22016)):
        Hh = F // 2
        out += [(tag, "fwd_qkv", M, q, d, 0, 0, EPI_BF16), (tag, "fwd_o", M, d, d, 0, 0, EPI_BF16),
                (tag, "fwd_gu", M, F, d, 0, 0, EPI_BF16), (tag, "fwd_down", M, d, Hh, 0, 0, EPI_RES),
                (tag, "dgrad_down", M, Hh, d, 0, 1, EPI_BF16), (tag, "dgrad_gu", M, d, F, 0, 1, EPI_BF16),
                (tag, "dgrad_o", M, d, d, 0, 1, EPI_BF16), (tag, "dgrad_qkv", M, d, q, 0, 1, EPI_BF16),
                (tag, "wgrad_down", d, Hh, M, 1, 1, EPI_ACC), (tag, "wgrad_gu", F, d, M, 1, 1, EPI_ACC),
                (tag, "wgrad_o", d, d, M, 1, 1, EPI_ACC), (tag, "wgrad_qkv", q, d, M, 1, 1, EPI_ACC),
                # first micro-step of an accumulation (GA = 1: every step): fresh bf16 epilogue
                (tag, "wgradF_down", d, Hh, M, 1, 1, EPI_BF16), (tag, "wgradF_gu", F, d, M, 1, 1, EPI_BF16),
                (tag, "wgradF_o", d, d, M, 1, 1, EPI_BF16), (tag, "wgradF_qkv", q, d, M, 1, 1, EPI_BF16)]
    return out


def child():
    import torch
    sys.path.insert(0, str(ROOT))
    from paper_2512_15306_b200 import ops
    res = []
    for tag, name, m, n, k, amn, bmn, epi in shapes():
        mk = lambda r, c: torch.randint(0, 120, (r, c), dtype=torch.uint8, device="cuda")
        a = mk(k, m) if amn else mk(m, k)
        b = mk(k, n) if bmn else mk(n, k)
        res_t = torch.zeros(m, n, dtype=torch.bfloat16, device="cuda") if epi == EPI_RES else None
        out = torch.zeros(m, n, dtype=torch.bfloat16, device="cuda")
        for bn in (0, 128, 256):
            kw = dict(M=m, N=n, K=k, a_mn=bool(amn), b_mn=bool(bmn), a_fmt=1 if bmn else 0, epi=epi, out=out,
                      res=res_t, sr=(1, 2, 3), bn=bn, split_k=0)
            try:
                plan = ops.gemm_plan(a, b, **kw)
                f = lambda: ops.gemm(a, b, **kw)
                f()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    f()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / 20 * 1e3
            except Exception as e:  # noqa: BLE001
                plan, us = {"error": str(e)[:80]}, None
            res.append({"shape": f"{tag}/{name}", "bn_req": bn, "plan": plan, "us": us,
                        "tflops": (2.0 * m * n * k / us / 1e6) if us else None})
    print(json.dumps(res))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        sys.exit(0)
    rows = {}
    for cg in ("0", "1", "2"):
        env = dict(os.environ, QTB_GEMM_CG=cg)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=900)
        if r.returncode:
            print(r.stderr[-2000:])
            continue
        for e in json.loads(r.stdout.strip().splitlines()[-1]):
            rows.setdefault(e["shape"], []).append((cg, e))
    for shape, lst in rows.items():
        print(shape)
        for cg, e in lst:
            p = e["plan"]
            if e["us"] is None:
                continue
            print(f"   force_cg={cg} bn_req={e['bn_req']:3d} -> cg={p['cg']} bn={p['bn']} splits={p['splits']} "
                  f"grid={p['grid']}  {e['us']:8.1f} us  {e['tflops']:7.1f} TF/s")
