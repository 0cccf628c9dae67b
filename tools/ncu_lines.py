"""Per-CUDA-source-line stall/instruction attribution from an ncu report (sass,cuda view)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, skip = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "--kernel-name", "regex:" + (sys.argv[3] if len(sys.argv) > 3 else "."), "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = None
st, ins = defaultdict(float), defaultdict(float)
text = {}
cur = None
for r in rows:
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < len(h):
        continue
    ln, src = r[0], r[1]
    if ln:
        cur = int(ln)
        text[cur] = src
    ws = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    try:
        st[cur] += float(r[ws] or 0)
        ins[cur] += float(r[ie] or 0)
    except ValueError:
        pass
ts, ti = sum(st.values()) or 1, sum(ins.values()) or 1
for ln, v in sorted(st.items(), key=lambda x: -x[1])[:30]:
    print(f"{100 * v / ts:5.1f}% stall {100 * ins[ln] / ti:5.1f}% inst  L{ln}: {text.get(ln, '')[:90]}")
