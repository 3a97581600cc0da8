#!/usr/bin/env python
"""Per-CUDA-source-line profile of one kernel from an ncu report (no GPU needed).

  python tools/ncu_lines.py report.ncu-rep k_sweep_a [top] [--ranges a-b:name,...] [--skip=i]
Prints instructions executed and warp-stall samples per source line (top lines),
the stall-reason mix, and optional line-range totals (kernel regions).
Needs a capture with --import-source on and a -lineinfo build.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 30
ranges = []
extra = []
for a in sys.argv[3:]:
    if a.startswith("--skip="):
        extra = ["--launch-skip", a.split("=", 1)[1], "--launch-count", "1"]
    if a.startswith("--ranges="):
        for part in a.split("=", 1)[1].split(","):
            lr, name = part.split(":")
            lo, hi = lr.split("-")
            ranges.append((int(lo), int(hi), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"] + extra, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
files = []
cur = None
lines = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iE = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if r and r[0] and r[0].isdigit():
        try:
            e = float(r[iE] or 0)
            s = float(r[iS] or 0)
        except (ValueError, IndexError):
            continue
        st = {}
        for i, h in stall_cols:
            try:
                st[h] = float(r[i] or 0)
            except ValueError:
                pass
        lines.append((cur, int(r[0]), r[1].strip(), e, s, st))
tot_e = sum(l[3] for l in lines) or 1
tot_s = sum(l[4] for l in lines) or 1
print(f"{kern}: {len(lines)} source lines, warp-instructions {tot_e:.4g}, stall samples {tot_s:.0f}")
mix = {}
for l in lines:
    for k, v in l[5].items():
        mix[k] = mix.get(k, 0) + v
print("stall mix:", ", ".join(f"{k[6:]}:{v / tot_s:.1%}" for k, v in sorted(mix.items(), key=lambda kv: -kv[1])[:10]))
print(f"top {top} lines by instructions (file:line  %inst  %stall  source):")
for l in sorted(lines, key=lambda l: -l[3])[:top]:
    f = l[0].split("/")[-1] if l[0] else "?"
    print(f"  {f}:{l[1]:<5d} {l[3] / tot_e:6.1%} {l[4] / tot_s:6.1%}  {l[2][:80]}")
print(f"top {top} lines by stall samples:")
for l in sorted(lines, key=lambda l: -l[4])[:top]:
    f = l[0].split("/")[-1] if l[0] else "?"
    st = sorted(l[5].items(), key=lambda kv: -kv[1])[:2]
    print(f"  {f}:{l[1]:<5d} {l[3] / tot_e:6.1%} {l[4] / tot_s:6.1%}  [{', '.join(k[6:] for k, _ in st)}] {l[2][:60]}")
for lo, hi, name in ranges:
    e = sum(l[3] for l in lines if lo <= l[1] <= hi and l[0] and l[0].endswith(".cu"))
    s = sum(l[4] for l in lines if lo <= l[1] <= hi and l[0] and l[0].endswith(".cu"))
    print(f"region {name:>14s} lines {lo}-{hi}: inst {e / tot_e:6.1%} stalls {s / tot_s:6.1%}")
