#!/usr/bin/env python
"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) into per-kernel
launch counts, mean and total time and share of the listed time (cold-cache,
serialised replays: the SHARE is what compares with the bench's live kernel times).

    python tools/launch_summary.py gpurun_out/launches_fin.csv profiles/r02s4_launches.md [title]
"""
import csv
import sys

src, dst = sys.argv[1], sys.argv[2]
title = sys.argv[3] if len(sys.argv) > 3 else "ncu launch list"
rows = list(csv.reader(open(src)))
hdr = None
per = {}
order = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("fbp::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
        if name not in per:
            per[name] = []
            order.append(name)
        per[name].append(us)
tot = sum(sum(v) for v in per.values())
lines = [f"# {title}", "", f"Source: `{src}` (ncu `--metrics gpu__time_duration.sum --clock-control none`).", "",
         "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
for n in order:
    v = per[n]
    lines.append(f"| `{n}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {sum(v) / tot:.3f} |")
open(dst, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
