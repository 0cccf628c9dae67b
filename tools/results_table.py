"""Markdown table of the committed bench lines (profiles/bench_<tag>_<config>.json
and their _n2 / _n4 scaling variants) for README.md / BASELINE.md.

usage: python tools/results_table.py [tag]   (default tag r2)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
NAMES = [("rmat20", "4: R-MAT S20 EF16, 65,536 sampled sources, 8192 per GPU per step (headline)"),
         ("rmat12", "1: R-MAT S12 EF16, all sources"),
         ("rmat16", "3: R-MAT S16 EF16, all sources, pruning off"),
         ("rmat16p", "3: same, pruning on (TEPS counts \\|S⁺\\|)"),
         ("grid", "2: grid 512×512, all sources (slices mode), 8192 per step"),
         ("rmat23", "5: R-MAT S23 EF16, 16,384 sampled sources, 2048 per GPU per step")]


def load(name):
    p = os.path.join(ROOT, "profiles", name)
    try:
        return json.load(open(p))
    except Exception:
        return None


rows = ["| Config (BASELINE.json) | GPUs | GTEPS | e2e GTEPS | ms / step | dominant kernel: frac of HBM (§8(d-iii)) | "
        "CPU oracle (host cores) |",
        "|---|---|---|---|---|---|---|"]
for cfg, label in NAMES:
    for suffix, n in (("", 1), ("_n2", 2), ("_n4", 4), ("_n8", 8)):
        d = load(f"bench_{tag}_{cfg}{suffix}.json")
        if not d:
            continue
        r = d.get("roofline") or {}
        kern = (r.get("kernel") or "").split(" ")[0]
        frac = r.get("frac")
        cpu = d.get("cpu_baseline") or {}
        e2e = d.get("e2e") or {}
        rows.append(f"| {label if n == 1 else ''} | {n} | {d['value'] / 1e9:.1f} | "
                    f"{(e2e.get('value') or 0) / 1e9:.1f} | {d['ms_per_step']:.2f} | "
                    f"{kern + f': {frac:.2f}' if frac is not None and n == 1 else ''} | "
                    f"{(str(round(cpu['value'] / 1e9, 2)) + ' G (' + str(cpu['cores']) + ' cores)') if cpu else ''} |")
print("\n".join(rows))
