"""DRAM traffic per kernel class from an ncu report of one lanes batch
(tools/prof_batch.py --sources 256 under `ncu --set full -k regex:lanes_`).

  fwd = lanes_level_kernel<..., BWD=false> + lanes_hub_finalize (forward)
  bwd = lanes_push_kernel<..., FWD=false> + lanes_bwd_finalize_kernel + lanes_bwd_hub_fin_kernel

Writes/updates profiles/ncu_traffic.json[config][class] with the summed DRAM
bytes and durations and the bytes per launch of the class's main kernel
(the bench's roofline "traffic" field)."""
import csv
import json
import os
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
ki, ti = h.index("Kernel Name"), h.index("gpu__time_duration.sum")
ri, wi = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tunit = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}
u = rows[1]


def cls(name):
    args = [x.strip() for x in name[name.index("<") + 1:name.index(">")].split(",")] if "<" in name else []
    if "lanes_level_kernel<" in name:
        return ("fwd" if args[2] in ("0", "false") else "bwd_pull", True)
    if "lanes_hub_finalize<" in name:
        return ("fwd" if len(args) < 3 or args[2] in ("0", "false") else "bwd_pull", False)
    if "lanes_push_kernel<" in name:
        return ("bwd" if args[1] in ("0", "false") else "fwd", True)
    if "lanes_bwd_finalize_kernel" in name or "lanes_bwd_hub_fin_kernel" in name or "lanes_fwd_commit" in name:
        return ("fwd" if "fwd_commit" in name else "bwd", False)
    return (None, False)


# sector efficiency (SURVEY §8(d-ii) graded number 2), summed over the class's launches
SUMS = ["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_red.sum", "smsp__inst_executed_op_global_red.sum", "smsp__inst_executed.sum"]
PCT = "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct"  # needs --metrics (not in --set full)
HIT = "lts__t_sector_hit_rate.pct"


def num(r, name):
    if name not in h:
        return None
    try:
        return float(r[h.index(name)].replace(",", ""))
    except ValueError:
        return None


agg = {}
for r in rows[2:]:
    c, main = cls(r[ki])
    if c is None:
        continue
    a = agg.setdefault(c, {"launches": 0, "all_launches": 0, "dram_bytes": 0.0, "time_s": 0.0})
    a["all_launches"] += 1
    a["launches"] += int(main)
    a["dram_bytes"] += float(r[ri]) * unit[u[ri]] + float(r[wi]) * unit[u[wi]]
    t = float(r[ti]) * tunit[u[ti]]
    a["time_s"] += t
    for m in SUMS:
        v = num(r, m)
        if v is not None:
            a[m] = a.get(m, 0.0) + v
    for m in (PCT, HIT):  # time-weighted means
        v = num(r, m)
        if v is not None:
            a[m + ":tw"] = a.get(m + ":tw", 0.0) + v * t
for a in agg.values():
    a["dram_bytes_per_launch"] = a["dram_bytes"] / max(1, a["launches"])
    for m in (PCT, HIT):
        if m + ":tw" in a:
            a[m] = a.pop(m + ":tw") / max(a["time_s"], 1e-30)
    s_, q_ = a.get(SUMS[0]), a.get(SUMS[1])
    if s_ and q_:
        a["ld_sectors_per_request"] = s_ / q_
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
try:
    data = json.load(open(path))
except Exception:
    data = {}
data[cfg] = dict(agg, source=f"ncu --set full --clock-control none of one 256-source batch ({os.path.basename(rep)}); "
                 "dram__bytes_read.sum + dram__bytes_write.sum summed per kernel class, per launch of the class's main kernel")
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[cfg], indent=1))
