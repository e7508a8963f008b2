#!/usr/bin/env python
"""Summarise the F1 ablation runs (scripts/gpu_run.sh ablation -> gpurun_out/ablation/*.json) as the shape
of the paper's tab:optimizations: speed-up of C (compact, reordering off), R (vanilla, reordered)
and C+R over the unoptimized U (vanilla, reordering off), training and inference, plus the
memory footprint (saved + scratch + graph index bytes, and the peak allocated)."""
import glob
import json
import os
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/abl"
rows = {}
for f in sorted(glob.glob(os.path.join(src, "*.json"))):
    try:
        d = json.load(open(f))
    except Exception:
        continue
    name = os.path.basename(f)[:-5]
    cfg, var = name.rsplit("_", 1)
    m = d["memory"]
    rows.setdefault(cfg, {})[var] = (d["ms_per_step"], m["saved_bytes"] + m["scratch_bytes"] + m["graph_index_bytes"],
                                     m["peak_allocated_bytes"], d["config"]["compaction_ratio"] if var in ("C", "CR") else None)
print("| workload | mode | U ms | C | R | C+R | compaction ratio | layer memory C+R / U | peak C+R / U (GB) |")
print("|---|---|---|---|---|---|---|---|---|")
for cfg in sorted(rows):
    v = rows[cfg]
    mode = "inference" if cfg.endswith("infer") else "training"
    wl = cfg[:-5] if cfg.endswith("infer") else cfg
    if "U" not in v:
        continue
    u = v["U"][0]
    sp = lambda k: ("%.2f" % (u / v[k][0])) if k in v else "n/a"
    best = "CR" if "CR" in v else "C"
    ratio = next((x[3] for x in v.values() if x[3] is not None), None)
    print(f"| {wl} | {mode} | {u:.3f} | {sp('C')} | {sp('R')} | {sp('CR')} | {ratio:.3f} | "
          f"{v[best][1] / v['U'][1]:.2f} | {v[best][2] / 1e9:.2f} / {v['U'][2] / 1e9:.2f} |")
