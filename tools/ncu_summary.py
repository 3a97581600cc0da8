#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py --launches gpurun_out/launches.csv \
         --report gpurun_out/prof.ncu-rep --out profiles/r01_<tag>.md [--json profiles/ncu_traffic.json]

* launches.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file` output;
  per-kernel launch count, mean duration and share of the libfbp kernel time.
* report: `ncu --set full -o` capture; per-kernel DRAM bytes, throughput,
  occupancy, shared-memory wavefronts, registers.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_cycles_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6,
              "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "second": 1.0}


def kind_of(name: str) -> str:
    for k, tag in (("k_iir", "iir"), ("k_fht_a", "fht_pass_a"), ("k_fht_b", "fht_pass_b"),
                   ("k_fht_pass_a", "fht_pass_a"), ("k_fht_pass_b", "fht_pass_b"),
                   ("k_sweep_a", "fht_pass_a"), ("k_sweep_ws", "fht_pass_a"), ("k_pair_b", "fht_pass_b")):
        if k in name:
            return tag
    return "other"


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[r[ki]].append(float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1e-9))
    return d


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        e = {"name": r[h.index("Kernel Name")]}
        for m, tag in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                e[tag] = v * UNIT_SCALE.get(units[i], 1.0)
        res.append(e)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--out", required=True)
    ap.add_argument("--json")
    # tools/gpu_cycle.sh's --set full capture runs `bench.py --batch ${NCU_FULL_BATCH:-2}`
    ap.add_argument("--slices-per-launch", type=float, default=2.0)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        d = launches(a.launches)
        fbp = {k: v for k, v in d.items() if kind_of(k) != "other"}
        tot = sum(sum(v) for v in fbp.values())
        lines += ["## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
                  "| kernel | launches | mean us | share of libfbp time |", "|---|---|---|---|"]
        for k, v in sorted(fbp.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k[:70]}` | {len(v)} | {1e6 * sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |")
        lines.append("")
    traffic = {}
    if a.report:
        rep = report(a.report)
        lines += ["## ncu --set full (per launch)", "",
                  "| kernel | us | DRAM read MB | DRAM write MB | DRAM % | SM % | occupancy % | smem wavefronts | FMA pipe % | L2 hit % | regs |",
                  "|---|---|---|---|---|---|---|---|---|---|---|"]
        per = collections.defaultdict(list)
        for e in rep:
            f = lambda k, s=1.0, fmt="{:.1f}": fmt.format(e[k] * s) if k in e else "-"
            lines.append(f"| `{e['name'][:50]}` | {f('time', 1e6)} | {f('dram_read', 1e-6)} | {f('dram_write', 1e-6)} | "
                         f"{f('dram_pct')} | {f('sm_pct')} | {f('occupancy_pct')} | {f('smem_wavefronts', 1.0, '{:.0f}')} | "
                         f"{f('fma_pipe_pct')} | {f('l2_hit_pct')} | {f('regs', 1.0, '{:.0f}')} |")
            per[kind_of(e["name"])].append(e)
        for k, es in per.items():
            rb = sum(e.get("dram_read", 0) + e.get("dram_write", 0) for e in es) / len(es)
            traffic[k] = {"dram_bytes_per_launch": rb, "dram_bytes_per_slice": rb / a.slices_per_launch,
                          "source": a.report}
        lines.append("")
    open(a.out, "w").write("\n".join(lines) + "\n")
    if a.json:
        json.dump(traffic, open(a.json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
