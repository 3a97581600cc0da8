#!/usr/bin/env python
"""Throughput of fbp_reconstruct at every BASELINE config (GPU, device-resident
inputs, CUDA events, 3 warm-ups), with the path roofline on SURVEY §8(d)'s 36 N^2
bytes per slice.  Writes a markdown table (argument: output path).

    python tools/measure_configs.py gpurun_out/r02_configs.md
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg  # noqa: E402
import phantoms as P  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
# (config, N, slices per call, distinct slices generated, steps)
CASES = [(1, 64, 4096, 64, 20), (2, 512, 256, 16, 20), (3, 2048, 1, 1, 50), (3, 2048, 16, 16, 20),
         (4, 1024, 256, 32, 10), (5, 4096, 8, 8, 10)]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    rows = []
    for cfg, N, B, G, K in CASES:
        c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_dc0.json")))
        plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
        S = torch.empty((B, 4, N, 2 * N), device="cuda")
        base = torch.stack([P.make_slice(cfg, i, device="cuda", N=N) for i in range(G)])
        for i in range(B):
            S[i] = base[i % G]
        del base
        img = torch.empty((B, N, N), device="cuda")
        for _ in range(3):
            plan.reconstruct(S, out=img)
        torch.cuda.synchronize()
        plan.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            plan.reconstruct(S, out=img)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        kt = plan.kernel_times()
        plan.profile(False)
        sps = B / (ms / 1e3)
        frac = 36.0 * N * N * sps / 1e9 / PEAK
        kms = ", ".join(f"{k} {v[0] / K:.3f}" for k, v in kt.items() if v[1])
        rows.append((cfg, N, B, plan.path()["fast"], ms, sps, frac, kms))
        print(rows[-1], flush=True)
        del S, img, plan
        torch.cuda.empty_cache()
    lines = ["| config | N | slices per call | fast path | ms per call | slices/s | path frac (36 N^2 B, measured HBM) | kernel ms per call |",
             "|---|---|---|---|---|---|---|---|"]
    for cfg, N, B, fast, ms, sps, frac, kms in rows:
        lines.append(f"| {cfg} | {N} | {B} | {fast} | {ms:.4f} | {sps:.1f} | {frac:.3f} | {kms} |")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if out:
        open(out, "w").write(txt)


if __name__ == "__main__":
    main()
