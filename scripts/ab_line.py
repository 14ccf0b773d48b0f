import json, sys
d = json.load(open(sys.argv[2]))
l = d["line"]
k = l["kernel_classes"]
print(sys.argv[1], round(l["value"]), round(l["ms_per_step"], 2), l["clocks"]["sm_mhz"],
      {c: k[c]["ms"] for c in ("gemm_fp8", "gemm_bf16", "attn_fwd", "attn_bwd", "ce_softmax", "elementwise") if c in k})
