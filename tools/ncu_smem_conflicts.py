#!/usr/bin/env python
"""Top shared-memory instructions by excessive (bank-conflict) wavefronts (no GPU).

  [NCU_INST=substring] python tools/ncu_smem_conflicts.py report.ncu-rep k_sweep_ws [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# several kernels (template instances) may match: keep the one whose full name
# contains $NCU_INST (default: the first)
inst = __import__("os").environ.get("NCU_INST", "")
blocks = []
for r in rows:
    if r and r[0] == "Kernel Name":
        blocks.append([r])
    elif blocks:
        blocks[-1].append(r)
rows = next(b for b in blocks if inst in b[0][1])
h = rows[1]
iS, iX, iW, iA = (h.index("Source"), h.index("L1 Wavefronts Shared Excessive"),
                  h.index("L1 Wavefronts Shared"), h.index("Address"))
data = []
for r in rows[2:]:
    try:
        data.append((float(r[iX] or 0), float(r[iW] or 0), r[iA], r[iS].strip()))
    except (ValueError, IndexError):
        pass
tx = sum(d[0] for d in data)
tw = sum(d[1] for d in data)
print(f"shared wavefronts {tw:.3e}, excessive {tx:.3e} ({100 * tx / max(tw, 1):.1f}%)")
for x, w, a, s in sorted(data, reverse=True)[:top]:
    print(f"{x:10.3e} {w:10.3e}  {a}  {s[:80]}")
