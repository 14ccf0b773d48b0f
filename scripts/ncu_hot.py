"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[si]) for r in rows[1:] if r[si].isdigit())
top = sorted((r for r in rows[1:] if r[si].isdigit()), key=lambda r: -int(r[si]))[:n]
print("total samples", tot)
for r in top:
    print(f"{int(r[si]):7d} {100*int(r[si])/tot:5.1f}%  {r[0][-5:]}  {r[1].strip()}")
