"""Top SASS instructions by warp-stall samples from an ncu --page source --csv --print-source sass export."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot)
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
idx = {d["Address"]: i for i, d in enumerate(data)}
for d in top:
    n = int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{n:7d} {100*n/tot:5.1f}%  [{idx[d['Address']]:5d}] {d['Source'].strip()[:90]}")
