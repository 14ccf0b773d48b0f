"""Top SASS lines by warp-stall samples from an ncu report (source page).
usage: ncu_hot.py REPORT [N] [KERNEL_REGEX]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
seen, uniq = set(), []
for r in rows[1:]:
    if r[si].isdigit() and r[0] not in seen:
        seen.add(r[0])
        uniq.append(r)
tot = sum(int(r[si]) for r in uniq)
print("total samples", tot)
for r in sorted(uniq, key=lambda r: -int(r[si]))[:n]:
    print(f"{int(r[si]):7d} {100*int(r[si])/tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
