#!/usr/bin/env python
"""Print the top warp-stall reasons per kernel of an ncu report (no GPU needed)."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:60])
    vals = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                vals.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("   " + ", ".join(f"{k}={v:.2f}" for v, k in sorted(vals, reverse=True)[:8]))
