#!/usr/bin/env python
"""Summarise an ncu --page details --csv export: per launch the key metrics (duration, DRAM / memory
throughput, L2 hit rate, occupancy, registers, eligible warps, stall cycles per issue)."""
import csv
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Eligible Warps Per Scheduler", "Issued Warp Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Compute (SM) Throughput", "Executed Ipc Active", "Block Limit Registers",
        "Dynamic Shared Memory Per Block", "Grid Size"]
path = sys.argv[1]
rows = list(csv.reader(open(path)))
h = rows[0]
ii, ki, mi, ui, vi = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
cur, seen = None, set()
print(f"# {path}: ncu --set full --clock-control none (cold-cache serialised replays; see DESIGN.md §6)")
for r in rows[1:]:
    if r[ii] != cur:
        cur = r[ii]
        seen = set()
        print(f"== [{r[ii]}] {r[ki][:150]}")
    if r[mi] in WANT and (r[mi], r[ui]) not in seen:
        seen.add((r[mi], r[ui]))
        print(f"   {r[mi]:<38} {r[vi]:>14} {r[ui]}")
