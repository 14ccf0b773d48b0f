"""Summarize an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys, collections, re
lines = [l for l in open(sys.argv[1]) if l.startswith("\"")]
rows = list(csv.DictReader(lines))
agg = collections.OrderedDict()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = re.sub(r"\(.*", "", name)
    m = re.search(r"gemm_kernel<(.*?)>", name)
    if m:
        short = "gemm<" + m.group(1) + ">"
    key = short + " grid" + r["Grid Size"]
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"]) / 1e3
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{us/1e3:9.3f} ms {100*us/tot:5.1f}%  n={n:4d}  avg {us/n:9.1f} us  {k}")
