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

Rank 0 prints ONE JSON line.  See DESIGN.md §7-8 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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


# ------------------------------------------------------------- rank logic
# (backend-agnostic; tests/test_bench_ranks.py drives it with gloo on CPU)
def rank_env():
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 without)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def slice_ids(rank: int, per_rank: int) -> list:
    """Distinct seeded slices per rank: rank r owns slices r*B .. r*B + B - 1."""
    return [rank * per_rank + i for i in range(per_rank)]


def time_steps(step, steps: int, barrier, sync, timer) -> float:
    """Barrier + sync, then exactly `steps` calls of step() between timer marks,
    sync + barrier.  timer() -> (start(), stop() -> ms)."""
    barrier()
    sync()
    start, stop = timer()
    start()
    for _ in range(steps):
        step()
    ms = stop()
    sync()
    barrier()
    return ms


def max_over_ranks(values, world: int, device="cpu"):
    """Element-wise max of per-rank timings (all_reduce MAX; identity at world 1)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def aggregate(world: int, per_rank: int, steps: int, max_ms: float) -> float:
    """Whole-job throughput: slices of all ranks / slowest rank's time."""
    return world * per_rank * steps / (max_ms / 1e3)


def cuda_timer(stream):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)

    def make():
        def start():
            e0.record(stream)

        def stop():
            e1.record(stream)
            e1.synchronize()
            return e0.elapsed_time(e1)
        return start, stop
    return make


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
def alg_bytes_per_slice(N: int) -> float:
    """read the 4 x N x 2N fp32 linogram, write the N x N fp32 image."""
    return 36.0 * N * N


def kernel_design_bytes(kind: str, N: int, NB: int, H: int, path: dict | None = None) -> float:
    """Bytes per SLICE each kernel's own contract must move, including
    the two-pass FHT's intermediate R; reported beside, not instead of, §8(d)."""
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
    """ncu DRAM bytes per slice of `kind` from the committed bench-batch capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    v = d.get(kind)
    if not isinstance(v, dict):
        return None, None
    return v.get("dram_bytes_per_slice"), v.get("source")


def path_dram(B: int, ms_step: float, world: int, peak: float):
    """ncu DRAM bytes per slice summed over the path's kernel kinds (profiles/
    ncu_traffic.json) x slices per step / live step time: SURVEY 8(d)'s ncu-achieved
    DRAM bandwidth, as a fraction of the measured peak and of 6557 / 8000 GB/s."""
    tot, src = 0.0, None
    for kind in ("fht_pass_a", "fht_pass_b"):
        b, s = ncu_traffic(kind)
        if b is None:
            return None
        tot += b
        src = s
    gbs = tot * B / (ms_step / 1e3) / 1e9
    return {"bytes_per_slice": tot, "achieved": gbs, "frac": gbs / peak, "frac_6557": gbs / 6557.0,
            "frac_8000": gbs / 8000.0, "unit": "GB/s per GPU", "source": src}


# ------------------------------------------------------- CPU oracle pool
_POOL_DATA = {}


def _pool_reconstruct(i):
    """Worker: the oracle on slice i % len(slices) (fork-inherited, untimed setup)."""
    from oracle import fbp_oracle as O
    S, b, a = _POOL_DATA["slices"][i % len(_POOL_DATA["slices"])], _POOL_DATA["b"], _POOL_DATA["a"]
    t0 = time.perf_counter()
    if _POOL_DATA.get("family") is None:
        O.reconstruct(S, b, a)
    else:
        import numpy as np
        f = (i + _POOL_DATA["family"]) % 4
        F = np.zeros_like(S)
        F[f] = O.iir_symmetric(S[f], b, a)
        O.combine(O.fht_backproject(F), 1.0 / S.shape[1])
    return time.perf_counter() - t0, time.time()


def host_cores():
    """(threads usable by this process, os.cpu_count(), CPU model)."""
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return usable, os.cpu_count(), model


def pool_workers(per_worker_gb: float) -> int:
    usable, _, _ = host_cores()
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE") / 2**30
        cap = max(1, int(0.6 * avail / per_worker_gb))
    except (ValueError, OSError):
        cap = usable
    return max(1, min(usable, cap))


class OraclePool:
    """The oracle as it stands, one single-threaded NumPy process per host core
    (fork start method: the seeded slices are inherited, not pickled)."""

    def __init__(self, slices, b, a, family=None, per_worker_gb=1.6):
        import multiprocessing as mp
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        _POOL_DATA.update(slices=slices, b=b, a=a, family=family)
        self.workers = pool_workers(per_worker_gb)
        self.pool = mp.get_context("fork").Pool(self.workers)

    def step(self, k: int = 0):
        """One round: every worker runs one task; returns the round's wall seconds."""
        t0 = time.time()
        res = self.pool.map(_pool_reconstruct, [k * self.workers + i for i in range(self.workers)],
                            chunksize=1)
        return max(r[1] for r in res) - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_baseline(slices_np, b, a):
    """Oracle throughput on a bounded sample of the same workload (rank 0, N=1):
    one full config-3 slice per host core, all in parallel."""
    usable, total, model = host_cores()
    pool = OraclePool(slices_np, b, a)
    dt = pool.step()
    w = pool.workers
    pool.close()
    return {"value": w / dt, "unit": UNIT, "cores": w, "kind": "oracle",
            "sample": f"{w} full config-3 slices (N=2048), one per process, NumPy fp64 oracle.reconstruct",
            "seconds": dt, "host_cpu_count": total, "affinity_cores": usable, "cpu_model": model}


# ---------------------------------------------------------------- arms
def run_reference(args):
    """The oracle as it stands, on the box's host cores (bench --impl reference)."""
    world, rank, _ = rank_env()
    if rank != 0:
        return
    import phantoms
    N = N_HEADLINE
    b, a = load_coeffs(N)
    slices = [phantoms.make_slice(CFG, i).double().numpy() for i in range(2)]
    # one step = one line family of one slice per host core (IIR on its N rows,
    # FHT back projection, its share of Eq.22), all cores in parallel
    pool = OraclePool(slices, b, a, family=0)
    for k in range(args.warmup):
        pool.step(k)
    dt = 0.0
    for k in range(args.steps):
        dt += pool.step(args.warmup + k)
    w = pool.workers
    pool.close()
    usable, total, model = host_cores()
    value = 0.25 * w * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config3: N=2048 slice, 4x2048x4096 linogram, 50-ellipse phantom",
                       "N": N, "step": f"one line family of one slice on each of {w} host processes "
                                       f"({0.25 * w:g} slices)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": w, "kind": "oracle",
                             "sample": f"{args.steps} steps x {w} quarter-slices (one family each) "
                                       "of config-3 slices 0-1", "host_cpu_count": total,
                             "affinity_cores": usable, "cpu_model": model},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_fbp(args):
    import torch
    import torch.distributed as dist
    import phantoms
    import paper_2007_06289_b200 as pkg
    from paper_2007_06289_b200 import dist as fdist

    world, rank, local = rank_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
        local = 0
    dev = torch.device(f"cuda:{local}")
    N = args.n
    b, a = load_coeffs(N, args.coeffs)
    B = args.batch
    plan = pkg.Plan(N, b, a, max_batch=B, device=local)
    info = plan.info()
    # distinct seeded slices per rank
    S = torch.empty((B, 4, N, 2 * N), device=dev, dtype=torch.float32)
    for i, sid in enumerate(slice_ids(rank, B)):
        S[i] = phantoms.make_slice(CFG, sid, device=dev, N=N)
    img = torch.empty((B, N, N), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def sync():
        torch.cuda.synchronize(dev)

    timer = cuda_timer(stream)
    launches = [0]

    def step():
        plan.reconstruct(S, out=img, stream=stream)

    def step_counted():
        step()
        launches[0] += plan.launch_count()

    for _ in range(max(args.warmup, 0)):
        step()
    sync()

    sampler = ClockSampler(local)
    sampler.start()
    plan.profile(True)
    ms = time_steps(step_counted, args.steps, barrier, sync, timer)
    ktimes = plan.kernel_times()
    plan.profile(False)
    # a clean (event-free) timing of the same K steps, for the headline value
    ms_clean = time_steps(step, args.steps, barrier, sync, timer)
    clocks = sampler.stop()
    ms_clean, ms = max_over_ranks([ms_clean, ms], world, dev)

    # ---- the SPEC plain-MSE coefficient set (beta != 0 sweep variant), same workload ----
    variants = {}
    if not args.no_variants and args.coeffs != "spec":
        bs, as_ = load_coeffs(N, "spec")
        plan_s = pkg.Plan(N, bs, as_, max_batch=B, device=local)
        for _ in range(3):
            plan_s.reconstruct(S, out=img, stream=stream)
        ks = max(3, min(args.steps, 20))
        plan_s.profile(True)
        ms_s = time_steps(lambda: plan_s.reconstruct(S, out=img, stream=stream), ks, barrier, sync, timer)
        kt_s = plan_s.kernel_times()
        plan_s.profile(False)
        ms_s = max_over_ranks([ms_s], world, dev)[0]
        variants["spec"] = {"value": aggregate(world, B, ks, ms_s), "unit": UNIT, "steps": ks,
                            "ms_per_step": ms_s / ks, "coeffs": "spec M=Q=3 (plain MSE fit, beta != 0)",
                            "schedule": plan_s.path(),
                            "kernel_ms_per_step": {k: v[0] / ks for k, v in kt_s.items() if v[1] > 0}}
        plan_s.close()
        del plan_s

    # ---- multi-GPU: gather every rank's images to rank 0 (NCCL), timed separately ----
    gather = None
    if world > 1 and not args.no_gather:
        n_total = world * B
        for _ in range(2):
            fdist.gather_volume(img, n_total, N, world, rank, dev)
        ms_g = time_steps(lambda: fdist.gather_volume(img, n_total, N, world, rank, dev), 3, barrier, sync,
                          timer)
        ms_g = max_over_ranks([ms_g], world, dev)[0] / 3
        gather = {"ms": ms_g, "bytes_to_rank0": (world - 1) * B * N * N * 4,
                  "GB_per_s_into_rank0": (world - 1) * B * N * N * 4 / (ms_g / 1e3) / 1e9,
                  "how": "torch.distributed.gather (NCCL) of [B, N, N] fp32 per rank to rank 0, "
                         "not in the headline timed region"}

    # ---- NEXT-1: forward FHT (fbp_fht_forward, Eq.17) of this step's images ----
    fwd = None
    if not args.no_forward:
        lin_f = torch.empty_like(S)
        for _ in range(3):
            plan.forward(img, out=lin_f, stream=stream)
        kf = max(1, min(args.steps, 20))
        plan.profile(True)
        ms_f = time_steps(lambda: plan.forward(img, out=lin_f, stream=stream), kf, barrier, sync, timer)
        kt_f = plan.kernel_times()
        plan.profile(False)
        ms_f = max_over_ranks([ms_f], world, dev)[0]
        alg_f = 36.0 * N * N                   # image read (4 N^2 B) + linogram write (32 N^2 B)
        fwd = {"value": aggregate(world, B, kf, ms_f), "unit": UNIT, "steps": kf, "ms_per_step": ms_f / kf,
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
        ms_r = time_steps(lambda: plan.resample(sino, dr=dr, out=lin_r, stream=stream), kr, barrier, sync,
                          timer)
        ms_r = max_over_ranks([ms_r], world, dev)[0]
        alg_r = 4.0 * na * nb + 32.0 * N * N        # sinogram read + linogram write
        rsm = {"value": aggregate(world, B, kr, ms_r), "unit": UNIT, "steps": kr, "ms_per_step": ms_r / kr,
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
        dt = max_over_ranks([dt], world, dev)[0]
        e2e = {"value": world * Be * reps / dt, "unit": UNIT,
               "h2d_bytes_per_step": Be * 4 * N * 2 * N * 4, "d2h_bytes_per_step": Be * N * N * 4,
               "slices_per_step": Be, "path": "fbp_reconstruct_host (pinned host buffers)"}

    if rank == 0:
        peak, peak_kind, _ = measured_peaks()
        value = aggregate(world, B, args.steps, ms_clean)
        # dominant kernel: SURVEY §8(d) algorithmic bytes (36 N^2 per slice) x the slices
        # one launch processes / its mean launch time (CUDA events on the launching stream)
        kinds = {k: v for k, v in ktimes.items() if v[1] > 0}
        dom = max(kinds, key=lambda k: kinds[k][0])
        dom_ms, dom_n = kinds[dom]
        per_step = dom_n / args.steps                     # launches of `dom` per step
        # pass B runs one launch per Eq.22 family pair, each over the same slices
        slices_per_launch = B / max(1.0, per_step / (2 if dom == "fht_pass_b" else 1))
        alg_launch = alg_bytes_per_slice(N) * slices_per_launch
        avg_launch_ms = dom_ms / dom_n
        achieved = alg_launch / (avg_launch_ms / 1e3) / 1e9
        design = kernel_design_bytes(dom, N, 1 << info["m"], 1 << info["k1"], plan.path())
        if dom == "fht_pass_b":
            design /= 2                                   # one launch = one family pair
        design_launch = design * slices_per_launch
        trf, trf_src = ncu_traffic(dom)
        if trf is not None:
            trf = trf * slices_per_launch / (2 if dom == "fht_pass_b" else 1)
        shares = {k: round(v[0] / max(ms, 1e-9), 4) for k, v in ktimes.items()}
        path_bytes = alg_bytes_per_slice(N) * world * B * args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_clean / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config3: N=2048 slices, 4x2048x4096 fp32 linogram each, "
                                   "seeded 50-ellipse phantoms (analytic line integrals)",
                       "N": N, "slices_per_gpu_per_step": B, "coeffs": f"{args.coeffs} M=Q=3",
                       "l2": f"inputs {B * 4 * N * 2 * N * 4 / 2**30:.1f} GiB/step per GPU > 126 MB L2 (no flush needed)",
                       "level_split": f"k1={info['k1']} m={info['m']}",
                       "schedule": plan.path(),
                       "parallelism": f"slices sharded over {world} GPU(s), no collective"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "alg_bytes_per_launch": alg_launch,
                         "alg_bytes": "SURVEY 8(d): 36 N^2 B per slice x slices per launch",
                         "avg_launch_ms": avg_launch_ms, "launches_per_step": per_step,
                         "traffic": trf, "traffic_source": trf_src,
                         "design_bytes_per_launch": design_launch,
                         "design_frac": design_launch / (avg_launch_ms / 1e3) / 1e9 / peak},
            "path_roofline": {"alg_bytes_per_slice": alg_bytes_per_slice(N),
                              "achieved": path_bytes / (ms_clean / 1e3) / 1e9 / world,
                              "frac": path_bytes / (ms_clean / 1e3) / 1e9 / world / peak,
                              "unit": "GB/s per GPU",
                              # SURVEY 8(d)'s other figure: ncu DRAM bytes of all kernels of
                              # one call (committed bench-batch capture) over the live step time
                              "ncu_dram": path_dram(B, ms_clean / args.steps, world, peak)},
            "kernel_share": shares,
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in ktimes.items()},
            "gpu_launches": launches[0],
            "clocks": clocks,
            "e2e": e2e,
        }
        if variants:
            line["variants"] = variants
        if gather:
            line["gather"] = gather
        nxt = {}
        for key, item in (("fht_forward", fwd), ("resample", rsm)):
            if item is not None:
                item["roofline"]["peak"] = peak
                item["roofline"]["frac"] = item["roofline"]["achieved"] / peak
                nxt[key] = item
        if nxt:
            line["next"] = nxt
        if world == 1 and not args.no_cpu_baseline:
            del S, img
            torch.cuda.empty_cache()
            slices_np = [phantoms.make_slice(CFG, i).double().numpy() for i in range(2)]
            line["cpu_baseline"] = cpu_baseline(slices_np, b, a)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 200; --impl reference: 10, each step ~2 s of oracle work)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=16, help="slices per GPU per step")
    ap.add_argument("--n", type=int, default=N_HEADLINE)
    ap.add_argument("--coeffs", default="dc0", choices=["dc0", "spec"])
    ap.add_argument("--impl", default="fbp", choices=["fbp", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-batch", type=int, default=8)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the spec-coefficient line")
    ap.add_argument("--no-gather", action="store_true")
    ap.add_argument("--no-forward", action="store_true", help="skip the NEXT-1/NEXT-2 line items (forward FHT, resampling)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 10 if args.impl == "reference" else 200
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_fbp(args)


if __name__ == "__main__":
    main()
