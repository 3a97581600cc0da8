#!/usr/bin/env python
"""Hot SASS regions of one kernel from an ncu report (no GPU needed).

  python tools/ncu_sass_hot.py report.ncu-rep k_iir [window]
Prints the instruction-count / stall-sample profile in windows of `window`
consecutive SASS instructions, plus the top single instructions by samples.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
win = int(sys.argv[3]) if len(sys.argv) > 3 else 64
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS, iE, iSamp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((r[iS].strip(), float(r[iE] or 0), float(r[iSamp] or 0)))
    except (ValueError, IndexError):
        pass
tot_e = sum(d[1] for d in data)
tot_s = sum(d[2] for d in data)
print(f"{len(data)} SASS instrs, executed {tot_e:.3g}, samples {tot_s:.0f}")
for i in range(0, len(data), win):
    seg = data[i:i + win]
    e = sum(d[1] for d in seg)
    s = sum(d[2] for d in seg)
    ops = {}
    for d in seg:
        op = d[0].split()[0] if d[0] else "?"
        if op.startswith("@"):
            op = d[0].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + d[1]
    top = ", ".join(f"{k}:{v / max(e, 1):.0%}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:5])
    print(f"[{i:5d}-{i + len(seg) - 1:5d}] exec {e / tot_e:6.1%} stalls {s / max(tot_s, 1):6.1%}  {top}")
print("top instructions by stall samples:")
for d in sorted(data, key=lambda d: -d[2])[:15]:
    print(f"  {d[2] / tot_s:6.1%}  exec {d[1]:.3g}  {d[0][:90]}")
