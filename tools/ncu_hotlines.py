"""Per-instruction view of one launch of an ncu report (source page, SASS):
instruction groups by execution count (per-hit / per-slot blocks) and the
hottest stall lines.  usage: python tools/ncu_hotlines.py REP KERNEL_REGEX LAUNCH_SKIP"""
import collections
import csv
import subprocess
import sys

rep, kre, skip = sys.argv[1], sys.argv[2], sys.argv[3]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
print(rows[0][:2])
h = rows[1]
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
iall, inot = h.index("Warp Stall Sampling (All Samples)"), h.index("Warp Stall Sampling (Not-issued Samples)")
seen, cnt, samp, lines = set(), collections.Counter(), collections.Counter(), []
for r in rows[2:]:
    if len(r) <= max(ia, iex, iall) or r[ia] in seen:
        continue
    seen.add(r[ia])
    try:
        ex, sa, ns = int(r[iex] or 0), int(r[iall] or 0), int(r[inot] or 0)
    except ValueError:
        continue
    cnt[ex] += 1
    samp[ex] += sa
    lines.append((sa, ns, ex, r[ia], r[isrc]))
tot = max(1, sum(x[0] for x in lines))
totx = max(1, sum(x[2] for x in lines))
print(f"warp instructions executed: {totx}")
print("instruction groups by execution count (instructions executed once per hit / per slot / ...):")
for ex, c in sorted(cnt.items(), key=lambda t: -t[0] * t[1])[:8]:
    print(f"  executed {ex:>12} times x {c:4d} instructions = {ex * c:>14} ({ex * c / totx * 100:4.1f} %), "
          f"stall samples {samp[ex] / tot * 100:5.1f} %")
print("hottest lines (all-samples %, not-issued %, executions, SASS):")
for x in sorted(lines, reverse=True)[:20]:
    print(f"  {x[0] / tot * 100:5.1f} % {x[1] / tot * 100:5.1f} % {x[2]:>10}  {x[4][:90]}")
