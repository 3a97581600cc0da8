#!/usr/bin/env python
"""Summarise a narrow-metric ncu capture at the bench batch (tools/gpu_prof.sh,
ncu16_<tag>.csv) into profiles/<name>.md and profiles/ncu_traffic.json (DRAM bytes
per slice of each kernel kind, the source of bench.py's roofline.traffic).

    python tools/ncu16_summary.py gpurun_out/ncu16_r2c.csv profiles/r02_ncu16.md [slices=16]
"""
import csv
import json
import os
import sys

src, dst = sys.argv[1], sys.argv[2]
slices = int(sys.argv[3]) if len(sys.argv) > 3 else 16
rows = list(csv.reader(open(src)))
hdr = None
k = {}
order = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        if key not in k:
            k[key] = {}
            order.append(key)
        k[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
lines = [f"# ncu narrow metrics at the bench batch ({slices} slices per launch, N = 2048)", "",
         f"Source: `{src}` (tools/gpu_prof.sh: `ncu --metrics ... --clock-control none -k regex:k_ -s 9 -c 3`",
         "on `bench.py --steps 1 --warmup 3 --batch 16`; replayed kernels, so times are per launch and",
         "serialised).  DRAM bytes per slice = launch bytes / slices.", "",
         "| kernel | us | DRAM read MB/slice | DRAM write MB/slice | DRAM TB/s | FMA pipe % | ALU pipe % | issue % | warps active % | L2 hit % | smem wavefronts/slice (M) |",
         "|---|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
for key in order:
    m = k[key]
    name = key[1].split("(")[0].replace("void ", "").replace("fbp::", "")
    us = m.get("gpu__time_duration.sum", 0) / 1e3
    rd = m.get("dram__bytes_read.sum", 0)
    wr = m.get("dram__bytes_write.sum", 0)
    lines.append(f"| `{name}` | {us:.1f} | {rd / slices / 1e6:.1f} | {wr / slices / 1e6:.1f} | "
                 f"{(rd + wr) / (us * 1e-6) / 1e12:.2f} | "
                 f"{m.get('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', float('nan')):.1f} | "
                 f"{m.get('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', float('nan')):.1f} | "
                 f"{m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', float('nan')):.1f} | "
                 f"{m.get('sm__warps_active.avg.pct_of_peak_sustained_active', float('nan')):.1f} | "
                 f"{m.get('lts__t_sector_hit_rate.pct', float('nan')):.1f} | "
                 f"{m.get('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 0) / slices / 1e6:.2f} |")
    kind = "fht_pass_a" if "sweep" in name else ("fht_pass_b" if "pair" in name else name)
    t = traffic.setdefault(kind, {"dram_bytes_per_slice": 0.0, "launches": 0})
    t["dram_bytes_per_slice"] += (rd + wr) / slices
    t["launches"] += 1
# whole path: ncu DRAM bytes over all kernels of one call / summed kernel time
tb = sum(k[key].get("dram__bytes_read.sum", 0) + k[key].get("dram__bytes_write.sum", 0) for key in order)
tt = sum(k[key].get("gpu__time_duration.sum", 0) for key in order) * 1e-9
if tt > 0:
    gbs = tb / tt / 1e9
    lines += ["", f"Whole path (all {len(order)} launches of one call): {tb / slices / 1e6:.1f} MB DRAM per slice, "
              f"{gbs:.0f} GB/s = {gbs / 6557:.3f} of 6557 GB/s (measured copy, SURVEY) / {gbs / 8000:.3f} of 8000 GB/s "
              f"(spec); algorithmic 36 N^2 = {36 * 2048 * 2048 / 1e6:.1f} MB per slice"]
for kind, t in traffic.items():
    t["source"] = os.path.basename(dst)
    t["batch"] = slices
with open(dst, "w") as fh:
    fh.write("\n".join(lines) + "\n")
json.dump(traffic, open(os.path.join(os.path.dirname(dst), "ncu_traffic.json"), "w"), indent=1)
print("\n".join(lines))
print(json.dumps(traffic, indent=1))
