"""Per-kernel share of the device time from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file F`):
launches, total and mean duration per kernel name, sorted by total."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':70s} {'launches':>9s} {'total ms':>10s} {'mean us':>9s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:70]:70s} {cnt[k]:9d} {v:10.3f} {1e3 * v / cnt[k]:9.2f} {100 * v / T:6.1f}%")
print(f"{'total':70s} {sum(cnt.values()):9d} {T:10.3f}")
