"""Summarise ncu --page raw --csv exports (units-aware): time, DRAM bytes, BW, SM/tensor utilisation."""
import csv, glob, sys
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "nsecond": 1e-9}
def load(f):
    rows = list(csv.reader(open(f)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            try:
                d[h] = float(v.replace(",", "")) * SCALE.get(u, 1)
            except ValueError:
                d[h] = v
        out.append(d)
    return out
for f in sorted(sys.argv[1:] or glob.glob("gpurun_out/ncu/*.raw.csv")):
    for d in load(f):
        t = d["gpu__time_duration.sum"]
        rb, wb = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        print(f"{str(d['Kernel Name'])[:48]:48s} grid={str(d.get('Grid Size',''))[:14]:14s} t={t*1e6:9.1f}us "
              f"rd={rb/1e6:9.1f}MB wr={wb/1e6:9.1f}MB {(rb+wb)/t/1e9:7.0f}GB/s sm%={d['sm__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f} "
              f"mem%={d['gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed']:5.1f} tensor%={d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0) or 0:5.1f} "
              f"warps%={d['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f} regs={d['launch__registers_per_thread']:.0f}")
