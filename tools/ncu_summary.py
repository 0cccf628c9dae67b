"""Summarise an ncu report: key SOL metrics, DRAM traffic, stall mix by opcode."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct"]
for r in rows[2:]:
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"  {k:70s} {r[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
for b in blocks:
    hh = b[0]
    si, ws, ie = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    tot = sum(float(r[ws] or 0) for r in b[1:]) or 1
    totie = sum(float(r[ie] or 0) for r in b[1:]) or 1
    op, opi = defaultdict(float), defaultdict(float)
    for r in b[1:]:
        s = r[si].strip()
        if s.startswith("@"):
            s = s.split(None, 1)[1] if " " in s else s
        o = (s.split()[0] if s else "").split(".")[0]
        op[o] += float(r[ws] or 0)
        opi[o] += float(r[ie] or 0)
    print("  stall/inst mix by opcode (top 14):")
    for o, v in sorted(op.items(), key=lambda x: -x[1])[:14]:
        print(f"    {o:10s} stall {100 * v / tot:5.1f}%  inst {100 * opi[o] / totie:5.1f}%")
    if len(sys.argv) > 2:
        items = sorted(((float(r[ws] or 0), i, r[si][:70], r[ie]) for i, r in enumerate(b[1:])), reverse=True)
        for s_, i, t, n in items[: int(sys.argv[2])]:
            print(f"    {100 * s_ / tot:5.1f}% {i:5d} {n:>12} {t}")
