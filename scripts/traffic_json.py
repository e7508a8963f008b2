#!/usr/bin/env python
"""ncu --page raw --csv of one step's traversal kernels -> profiles/ncu_traffic.json (DRAM read+write bytes
per bench kernel label, per step).  Usage: traffic_json.py raw.csv config [out.json]"""
import csv
import json
import sys

LABELS = [("k_hgt_bwd_pair", "hgt_bwd_pair"), ("k_hgt_bwd_dst", "hgt_bwd_dst"), ("k_hgt_fwd", "hgt_fwd_traverse"),
          ("k_rgat_bwd_pair", "rgat_bwd_pair"), ("k_rgat_bwd_dst", "rgat_bwd_dst"), ("k_rgat_fwd", "rgat_fwd_traverse"),
          ("k_rgcn_bwd_pair", "rgcn_bwd_pair"), ("k_rgcn_fwd", "rgcn_fwd_traverse")]
path, cfg = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
rows = list(csv.reader(open(path)))
h, units = rows[0], rows[1]
ki, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = {}
for r in rows[2:]:
    name = r[ki]
    lab = next((l for k, l in LABELS if k in name), None)
    if lab is None:
        continue
    b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
    per.setdefault(lab, 0.0)
    per[lab] += b
try:
    js = json.load(open(out))
except (OSError, ValueError):
    js = {}
js[cfg] = {k: {"bytes_per_step": int(v)} for k, v in per.items()}
js["_source"] = ("ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of the label's launches in one step "
                 "(warp, group and short halves summed): profiles/r01_ncu_traversal_*.txt")
json.dump(js, open(out, "w"), indent=1)
print(json.dumps(js[cfg]))
