"""Per-kernel duration, issue stats and top warp-stall reasons from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[0]
keys = ["gpu__time_duration.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:60]
    print(name)
    for k in keys:
        for i, c in enumerate(h):
            if c == k:
                print(f"   {k} = {r[i]}")
    st = [(h[i], r[i]) for i in range(len(h)) if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
    st = sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:8]
    print("   stalls:", ", ".join(f"{k.split('stalled_')[1]}={v}" for k, v in st))
