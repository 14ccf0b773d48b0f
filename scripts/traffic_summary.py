"""Per-kernel-class DRAM traffic of one training step from an ncu metrics CSV
(dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum per launch).
Classes follow bench.py's kernel_classes.  Writes profiles/<tag>_traffic.json."""
import collections, csv, json, re, sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}


def klass(name):
    m = re.search(r"gemm_kernel<(\d+),", name)
    if m:
        return "gemm_fp8" if m.group(1) == "0" else "gemm_bf16"
    for pat, c in (("splitk_reduce", "gemm_fp8"), ("quantize|absmax", "quant"), ("rms|colsum", "rmsnorm"),
                   ("fwd_tc_kernel|fwd1_tc|fwd1p_tc|attn::fwd_kernel", "attn_fwd"), ("dq_tc|dkdv_tc|bwd_dot|bwd_dq|bwd_dkdv", "attn_bwd"),
                   ("ce_softmax|loss_reduce", "ce_softmax"), ("adamw", "adamw"), ("norm_partials|sum_f64", "grad_norm")):
        if re.search(pat, name):
            return c
    return "elementwise"


rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
recs = collections.defaultdict(dict)
for r in csv.DictReader(rows):
    try:
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1)
    except ValueError:
        continue
    recs[r["ID"]][r["Metric Name"]] = v
    recs[r["ID"]]["name"] = r["Kernel Name"]
agg = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "time_s": 0.0})
for r in recs.values():
    a = agg[klass(r["name"])]
    a["launches"] += 1
    a["dram_bytes"] += r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
    a["time_s"] += r.get("gpu__time_duration.sum", 0)
out = {k: {"launches": v["launches"], "dram_bytes_per_launch": v["dram_bytes"] / v["launches"],
           "dram_gbs": v["dram_bytes"] / max(v["time_s"], 1e-12) / 1e9, "ncu_ms": v["time_s"] * 1e3}
       for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["time_s"])}
json.dump({"source": sys.argv[1], "note": "ncu serialised replay (cold L2 per launch); per-launch DRAM bytes",
           "classes": out}, open(sys.argv[2], "w"), indent=1)
for k, v in out.items():
    print(f"{k:12s} n={v['launches']:5d} {v['dram_bytes_per_launch']/1e6:10.1f} MB/launch {v['dram_gbs']:8.0f} GB/s {v['ncu_ms']:8.2f} ms")
