#!/usr/bin/env python
"""Benchmark: N x N fp32 slices/s at N = 2048 (BASELINE config 3), 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl fbp|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one process per GPU)

A step = one fbp_reconstruct (IIR ramp filter + FHT back projection, the whole
hot path) over a batch of B distinct seeded N=2048 linograms resident in HBM on
each rank (weak scaling: B slices per GPU, no collective on the data path).
Timing: W warm-up steps, barrier + synchronize, CUDA events on the launching
stream around exactly K steps, max over ranks.  Inputs (B x 128 MiB) exceed the
126 MB L2, so no flush is needed between steps.

Rank 0 prints ONE JSON line.  See DESIGN.md §8 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = 3
N_HEADLINE = 2048
METRIC = "N×N fp32 slices/sec (N=2048)"
UNIT = "slices/s"


def load_coeffs(N, variant="dc0"):
    c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_{variant}.json")))
    return c["b"], c["a"]


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback", 1965.0


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join("/tmp", f"fbp_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        self.t0 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), power=float(parts[3]),
                                 hw=parts[5], hwt=parts[6], swt=parts[7], pcap=parts[8]))
            except ValueError:
                continue
        if not rows:
            return None
        load = [r for r in rows if r["power"] > 200.0] or rows
        reasons = set()
        for r in load:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"),
                            ("swt", "sw_thermal_slowdown"), ("pcap", "sw_power_cap")):
                if r[k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in load),
                "sm_max_mhz": max(r["smax"] for r in load), "reasons": sorted(reasons),
                "samples": len(load), "power_w_max": max(r["power"] for r in load)}


# --------------------------------------------------------------- roofline
def kernel_algorithmic_bytes(kind: str, N: int, NB: int, H: int, path: dict | None = None) -> float:
    """Algorithmic HBM bytes per SLICE of each kernel."""
    W = 2 * N
    lin = 4.0 * N * W * 4                                  # 32 N^2 B
    # compact pass-A output: per family sum_b H rows of (N + b) floats
    r_fam = sum(H * (N + b) for b in range(NB)) * 4.0
    img = 4.0 * N * N
    if kind == "iir":
        return 2 * lin                                     # read S, write F
    if kind == "fht_pass_a":
        if path and path.get("fast"):
            # fused sweep: reads rows of block b from tile max(0, j0(b) - D), writes R
            X, D = path["tile_width"], path["lookahead_tiles"]
            nt = W // X
            cols = sum((nt - max(0, (N - (b + 1) * H + 1) // X - D)) * X for b in range(NB))
            return 4.0 * H * cols * 4 + 4 * r_fam
        return lin + 4 * r_fam                             # read F, write R
    if kind == "fht_pass_b":
        return 4 * r_fam + img + 2 * img                   # read R; write v-pair, RMW h-pair
    raise KeyError(kind)


def ncu_traffic(kind: str):
    """DRAM bytes per launch of `kind` from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = d.get(kind)
    return v.get("dram_bytes_per_slice") if isinstance(v, dict) else None


# ---------------------------------------------------------------- arms
def run_reference(args):
    """The oracle as it stands, on host cores (bench --impl reference)."""
    import numpy as np
    import torch
    import phantoms
    from oracle import fbp_oracle as O
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N = N_HEADLINE
    b, a = load_coeffs(N)
    # one step = the oracle on one line family of one slice (IIR on its N rows,
    # FHT back projection, its share of Eq.22): a bounded quarter-slice sample.
    S = phantoms.make_slice(CFG, 0).double().numpy()
    def step(f):
        F = O.iir_symmetric(S[f], b, a)
        Ff = np.zeros((4, N, 2 * N))
        Ff[f] = F
        return O.combine(O.fht_backproject(Ff), 1.0 / N)
    for i in range(args.warmup):
        step(i % 4)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i % 4)
    dt = time.perf_counter() - t0
    value = 0.25 * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config3: N=2048 slice, 4x2048x4096 linogram, 50-ellipse phantom",
                       "N": N, "step": "one line family of one slice (0.25 slice)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} quarter-slices (one family each) of config-3 slice 0"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(N, b, a, budget_s=25.0):
    """Oracle on a bounded sample of the same workload, rank 0 at N=1."""
    import phantoms
    from oracle import fbp_oracle as O
    S = phantoms.make_slice(CFG, 0).double().numpy()
    t0 = time.perf_counter()
    O.reconstruct(S, b, a)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": "1 full config-3 slice (N=2048) through oracle.reconstruct, NumPy fp64, 1 thread",
            "seconds": dt}


def run_fbp(args):
    import torch
    import torch.distributed as dist
    import phantoms
    import paper_2007_06289_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
        local = 0
    dev = torch.device(f"cuda:{local}")
    N = args.n
    b, a = load_coeffs(N)
    B = args.batch
    plan = pkg.Plan(N, b, a, max_batch=B, device=local)
    info = plan.info()
    # distinct seeded slices per rank: slice index rank*B + i
    S = torch.empty((B, 4, N, 2 * N), device=dev, dtype=torch.float32)
    for i in range(B):
        S[i] = phantoms.make_slice(CFG, rank * B + i, device=dev, N=N)
    img = torch.empty((B, N, N), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        plan.reconstruct(S, out=img, stream=stream)
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    torch.cuda.synchronize(dev)
    plan.profile(True)
    launches = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.reconstruct(S, out=img, stream=stream)
        launches += plan.launch_count()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    ms = e0.elapsed_time(e1)
    ktimes = plan.kernel_times()
    plan.profile(False)
    # a clean (event-free) timing of the same K steps, for the headline value
    torch.cuda.synchronize(dev)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        plan.reconstruct(S, out=img, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    ms_clean = e0.elapsed_time(e1)
    clocks = sampler.stop()

    t = torch.tensor([ms_clean, ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_clean, ms = float(t[0]), float(t[1])

    # ---- NEXT-1: forward FHT (fbp_fht_forward, Eq.17) of this step's images ----
    fwd = None
    if not args.no_forward:
        lin_f = torch.empty_like(S)
        for _ in range(3):
            plan.forward(img, out=lin_f, stream=stream)
        kf = max(1, min(args.steps, 20))
        torch.cuda.synchronize(dev)
        barrier()
        plan.profile(True)
        e0.record(stream)
        for _ in range(kf):
            plan.forward(img, out=lin_f, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms_f = e0.elapsed_time(e1)
        kt_f = plan.kernel_times()
        plan.profile(False)
        tf = torch.tensor([ms_f], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tf, op=dist.ReduceOp.MAX)
        ms_f = float(tf[0])
        alg_f = 36.0 * N * N                   # image read (4 N^2 B) + linogram write (32 N^2 B)
        fwd = {"value": world * B * kf / (ms_f / 1e3), "unit": UNIT, "steps": kf, "ms_per_step": ms_f / kf,
               "input": "this step's reconstructed images", "gpu_launches_per_step": plan.launch_count(),
               "kernel_ms_per_step": {k: v[0] / kf for k, v in kt_f.items() if v[1] > 0},
               "roofline": {"bound": "hbm", "alg_bytes_per_slice": alg_f, "unit": "GB/s per GPU",
                            "achieved": alg_f * B * kf / (ms_f / 1e3) / 1e9}}
        del lin_f

    # ---- NEXT-2: sinogram -> linogram resampling (fbp_resample_sinogram, Eq.14-15) ----
    rsm = None
    if not args.no_forward:
        import math
        na, dr = 2 * N, 1.0
        nb = int(math.ceil(math.sqrt(2) * N / dr)) + 4
        E = phantoms.draw_ellipses(N, 50, (N / 128, N / 3.2), seed=1000 * CFG + rank * B)
        sino1 = phantoms.sinogram_of_ellipses(E, N, na, nb, dr).to(torch.float32).to(dev)
        sino = sino1.unsqueeze(0).repeat(B, 1, 1).contiguous()
        del sino1
        lin_r = torch.empty_like(S)
        for _ in range(3):
            plan.resample(sino, dr=dr, out=lin_r, stream=stream)
        kr = max(1, min(args.steps, 20))
        torch.cuda.synchronize(dev)
        barrier()
        e0.record(stream)
        for _ in range(kr):
            plan.resample(sino, dr=dr, out=lin_r, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms_r = e0.elapsed_time(e1)
        tr = torch.tensor([ms_r], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        ms_r = float(tr[0])
        alg_r = 4.0 * na * nb + 32.0 * N * N        # sinogram read + linogram write
        rsm = {"value": world * B * kr / (ms_r / 1e3), "unit": UNIT, "steps": kr, "ms_per_step": ms_r / kr,
               "input": f"analytic 50-ellipse sinogram, {na} angles x {nb} bins, dr={dr}",
               "gpu_launches_per_step": plan.launch_count(),
               "roofline": {"bound": "hbm", "alg_bytes_per_slice": alg_r, "unit": "GB/s per GPU",
                            "achieved": alg_r * B * kr / (ms_r / 1e3) / 1e9}}
        del lin_r, sino

    # ---- end to end through the public host-buffer C-ABI call ----
    e2e = None
    if not args.no_e2e:
        Be = min(B, args.e2e_batch)
        host_in = S[:Be].cpu().pin_memory()
        host_out = torch.empty((Be, N, N), dtype=torch.float32).pin_memory()
        plan.reconstruct_host(host_in, out=host_out)      # warm (allocates staging)
        barrier()
        t0 = time.perf_counter()
        reps = max(1, args.e2e_steps)
        for _ in range(reps):
            plan.reconstruct_host(host_in, out=host_out)
        dt = time.perf_counter() - t0
        te = torch.tensor([dt], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dt = float(te[0])
        e2e = {"value": world * Be * reps / dt, "unit": UNIT,
               "h2d_bytes_per_step": Be * 4 * N * 2 * N * 4, "d2h_bytes_per_step": Be * N * N * 4,
               "slices_per_step": Be, "path": "fbp_reconstruct_host (pinned host buffers)"}

    if rank == 0:
        peak, peak_kind, _ = measured_peaks()
        total = world * B * args.steps
        value = total / (ms_clean / 1e3)
        # dominant kernel
        kinds = {k: v for k, v in ktimes.items() if v[1] > 0}
        dom = max(kinds, key=lambda k: kinds[k][0])
        dom_ms, dom_n = kinds[dom]
        slices_per_launch = (B * args.steps) / dom_n if dom != "fht_pass_b" else (B * args.steps) / (dom_n / 2)
        alg = kernel_algorithmic_bytes(dom, N, 1 << info["m"], 1 << info["k1"], plan.path())
        if dom == "fht_pass_b":
            alg = alg / 2                     # one launch = one family pair
        per_launch_bytes = alg * slices_per_launch
        achieved = per_launch_bytes / (dom_ms / dom_n / 1e3) / 1e9
        trf = ncu_traffic(dom)
        if trf is not None:
            trf = trf * slices_per_launch               # per launch, like `achieved`
        shares = {k: round(v[0] / max(ms, 1e-9), 4) for k, v in ktimes.items()}
        path_bytes = 36.0 * N * N * total
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_clean / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config3: N=2048 slices, 4x2048x4096 fp32 linogram each, "
                                   "seeded 50-ellipse phantoms (analytic line integrals)",
                       "N": N, "slices_per_gpu_per_step": B, "coeffs": "dc0 M=Q=3",
                       "l2": f"inputs {B * 4 * N * 2 * N * 4 / 2**30:.1f} GiB/step per GPU > 126 MB L2 (no flush needed)",
                       "level_split": f"k1={info['k1']} m={info['m']}",
                       "schedule": plan.path(),
                       "parallelism": f"slices sharded over {world} GPU(s), no collective"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": trf, "alg_bytes_per_launch": per_launch_bytes,
                         "avg_launch_ms": dom_ms / dom_n},
            "path_roofline": {"alg_bytes_per_slice": 36.0 * N * N,
                              "achieved": path_bytes / (ms_clean / 1e3) / 1e9 / world,
                              "frac": path_bytes / (ms_clean / 1e3) / 1e9 / world / peak,
                              "unit": "GB/s per GPU"},
            "kernel_share": shares,
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in ktimes.items()},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
        }
        nxt = {}
        for key, item in (("fht_forward", fwd), ("resample", rsm)):
            if item is not None:
                item["roofline"]["peak"] = peak
                item["roofline"]["frac"] = item["roofline"]["achieved"] / peak
                nxt[key] = item
        if nxt:
            line["next"] = nxt
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(N, b, a)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=16, help="slices per GPU per step")
    ap.add_argument("--n", type=int, default=N_HEADLINE)
    ap.add_argument("--impl", default="fbp", choices=["fbp", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-batch", type=int, default=8)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-forward", action="store_true", help="skip the NEXT-1/NEXT-2 line items (forward FHT, resampling)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_fbp(args)


if __name__ == "__main__":
    main()
