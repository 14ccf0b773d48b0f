"""Measured FP8 dense peak on this B200 (the roofline denominator MEASURED_PEAKS.json
lacks): the product's tcgen05 FP8 GEMM (qtk_gemm, E4M3 x E4M3 -> bf16) and
cuBLASLt's FP8 GEMM (torch._scaled_mm) at 8192^3, best-of-10 (burst) and
back-to-back for ~3 s (sustained), CUDA events on the launching stream.
Writes profiles/fp8_gemm_peak.json."""
import json
import pathlib
import sys
import time

import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2512_15306_b200 import ops  # noqa: E402

N = 8192
flops = 2.0 * N ** 3


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


def measure(fn):
    for _ in range(5):
        fn()
    burst = max(flops / timed(fn, 1) for _ in range(10)) / 1e12
    t0 = time.time()
    n = 0
    tot = 0.0
    while time.time() - t0 < 3.0:
        tot += timed(fn, 20) * 20
        n += 20
    return burst, flops * n / tot / 1e12


a = (torch.randn(N, N, device="cuda") * 0.5).to(torch.bfloat16)
b = (torch.randn(N, N, device="cuda") * 0.5).to(torch.bfloat16)
sa, sb = ops.absmax(a), ops.absmax(b)
ac, asc = ops.quantize(a, 0, sa)
bc, bsc = ops.quantize(b, 0, sb)
out = torch.empty(N, N, dtype=torch.bfloat16, device="cuda")
ours = measure(lambda: ops.gemm(ac, bc, M=N, N=N, K=N, a_scale=asc, b_scale=bsc, out=out))
res = {"shape": [N, N, N], "ours_tflops_burst": ours[0], "ours_tflops_sustained": ours[1]}
try:
    a8 = a.to(torch.float8_e4m3fn)
    b8 = b.to(torch.float8_e4m3fn).t()
    one = torch.ones((), device="cuda")
    cub = measure(lambda: torch._scaled_mm(a8, b8, scale_a=one, scale_b=one, out_dtype=torch.bfloat16))
    res.update({"cublaslt_tflops_burst": cub[0], "cublaslt_tflops_sustained": cub[1]})
except Exception as e:  # noqa: BLE001
    res["cublaslt_error"] = str(e)[:200]
best = max(res.get("ours_tflops_burst", 0), res.get("cublaslt_tflops_burst", 0))
res["tflops"] = best
res["how"] = ("max over the product's tcgen05 FP8 GEMM and cuBLASLt FP8 (torch._scaled_mm) of the best-of-10 "
              f"{N}^3 E4M3 GEMM time (2*N^3 flops), CUDA events; sustained = back-to-back for 3 s")
print(json.dumps(res, indent=1))
out_p = ROOT / "profiles" / "fp8_gemm_peak.json"
out_p.write_text(json.dumps(res, indent=1) + "\n")
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "fp8_gemm_peak.json").write_text(json.dumps(res, indent=1) + "\n")
