#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of `bench.py --steps S --warmup W`:
per kernel name the launches, total and mean duration, and the share of the layer step (kernels launched a
multiple of S+W times; one-off graph-build kernels are listed separately)."""
import collections
import csv
import sys

path, per = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 5
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mn = h.index("Metric Name") if "Metric Name" in h else None
tot, cnt = collections.defaultdict(float), collections.Counter()
dram = collections.defaultdict(float)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    name = r[mn] if mn is not None else "gpu__time_duration.sum"
    if name.startswith("dram__bytes"):  # optional DRAM read / write bytes of the same launches
        dram[r[kn]] += float(r[mv].replace(",", "")) * bscale.get(r[mu], 1.0)
        continue
    if name != "gpu__time_duration.sum":
        continue
    tot[r[kn]] += float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
    cnt[r[kn]] += 1
step = {k: v for k, v in tot.items() if cnt[k] % per == 0}
T = sum(step.values())
print(f"# {path}: ncu gpu__time_duration.sum per launch (--clock-control none; cold-cache, serialised launches:")
print(f"# compare SHARES, not absolutes).  Per-step kernels = launched a multiple of {per} times (warm-up + timed steps + the per-kernel profiling pass of bench.py).")
print(f"{'share':>7} {'launches':>8} {'mean us':>10} {'total us':>11} {'DRAM GB/launch':>14} {'DRAM TB/s':>9}  kernel")
for k, v in sorted(step.items(), key=lambda x: -x[1]):
    gb = dram[k] / cnt[k] / 1e9 if k in dram else float("nan")
    tbs = dram[k] / (v * 1e-6) / 1e12 if k in dram and v > 0 else float("nan")
    print(f"{100 * v / T:6.2f}% {cnt[k]:8d} {v / cnt[k]:10.1f} {v:11.1f} {gb:14.3f} {tbs:9.2f}  {k[:110]}")
print("# one-off (graph build, plans):")
for k, v in sorted(((k, v) for k, v in tot.items() if k not in step), key=lambda x: -x[1]):
    print(f"{'':7} {cnt[k]:8d} {v / cnt[k]:10.1f} {v:11.1f}  {k[:110]}")
