#!/usr/bin/env python
"""bench.py -- FP64 SEM Ax+gs and Jacobi-PCG throughput on 1..8 B200 (one process per GPU).

Metric (BASELINE.json): "FP64 Ax+gs GDOF/s and PCG iter/s at N=7, 1/2/4/8 B200,
% of HBM roofline".  A STEP is one nek_pcg_solve of 100 fixed Jacobi-PCG
iterations (every row of SURVEY 8(a) on the path: Ax, local gather-scatter, the
halo exchange when N>1, the mask, the fused CG updates and dot-product
reductions).  `value` is the BP5-style throughput of the whole job:
    value = sum over ranks of n_dof * iterations / max-over-ranks device time,
n_dof = E * N^3, in GDOF/s; pcg_iter_per_s = value / n_dof_total.
Ax+gs GDOF/s (nek_ax alone) is reported in `ax_gs`.

Workload at N=1: BASELINE configs[1] = 16^3 elements, N=7, bubble-deformed unit
box, Dirichlet on all faces, Poisson (h1,h2) = (1,0), b = seeded smooth field.
N>1: weak scaling, each rank owns one 16^3 z-slab of a 16 x 16 x 16N box.
Inputs are resident in HBM when the timed region starts; L2 (126 MiB) is
flushed between timed steps by writing a 256 MiB buffer (outside the events).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
       (N>1 via: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# keep stdout to the one JSON line (NCCL prints a version banner at some debug levels)
os.environ.setdefault("NCCL_DEBUG", "WARN")

METRIC = "FP64 Ax+gs GDOF/s and PCG iter/s at N=7, 1/2/4/8 B200, % of HBM roofline"
ITERS = 100
EX = EY = EZ_PER_RANK = 16
NORD = 7


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iters", type=int, default=ITERS)
    ap.add_argument("--ez", type=int, default=EZ_PER_RANK, help="element layers per rank")
    ap.add_argument("--order", type=int, default=NORD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pmg", action="store_true", help="skip the Jacobi vs pMG time-to-solution section")
    ap.add_argument("--no-peaks", action="store_true", help="skip the on-box peak probes")
    ap.add_argument("--no-beyond", action="store_true", help="skip the beyond-L2 roofline point (16x16x128)")
    ap.add_argument("--variant", type=int, default=0, help="Ax kernel variant (nek_set_variant; 0 = default)")
    ap.add_argument("--mesh", default="box", choices=["box", "rod", "cfg3"],
                    help="box: 16x16xez elements per GPU (config 2 at ez=16); rod: 17x17-pin rod bundle, "
                         "--rod-layers element layers per GPU (config 4 at 3 layers)")
    ap.add_argument("--rod-layers", type=int, default=3)
    ap.add_argument("--h2", type=float, default=0.0, help="Helmholtz mass coefficient (0 = Poisson)")
    ap.add_argument("--graph", action="store_true", help="no per-kernel event nodes in the CUDA graph "
                    "(no per-replay synchronisation; no roofline then)")
    return ap.parse_args()


def rank_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_mesh(rank, world, ez, N, args=None):
    from workloads import meshgen as mg
    if args is not None and args.mesh == "rod":
        L = args.rod_layers
        return mg.rod_bundle(17, 17, L, N, dirichlet="pins_walls" if args.h2 != 0.0 else "outlet",
                             z0_layer=rank * L, nlayers_total=L * world)
    if args is not None and args.mesh == "cfg3":
        # BASELINE config 3: E = 32 x 64 x 64 = 131072 (~45M DOF) fixed, z-slabs of 64/P layers (strong scaling)
        if 64 % world:
            raise SystemExit("cfg3 needs a rank count dividing 64")
        lz = 64 // world
        return mg.box_mesh(32, 64, 64, N, deform="bubble", eps=0.05, dirichlet="all",
                           zlayers=(rank * lz, (rank + 1) * lz))
    # every rank owns a unit cube of 16 x 16 x ez elements (cubic elements at any rank count: the per-GPU
    # problem of weak scaling does not change shape with N; at N = 1, ez = 16 this is config 2)
    return mg.box_mesh(EX, EY, ez * world, N, deform="bubble", eps=0.05, dirichlet="all",
                       extent=(1.0, 1.0, ez * world / float(EX)), zlayers=(rank * ez, (rank + 1) * ez))


def workload_name(args, world):
    kind = "Helmholtz (h1,h2)=(1,%g)" % args.h2 if args.h2 != 0.0 else "Poisson"
    if args.mesh == "cfg3":
        return (f"SEM {kind} Jacobi-PCG, {args.iters} iters/step; config 3: bubble-deformed box 32x64x64 elements "
                f"(E = 131072, ~45M DOF) split into {world} z-slab(s), N={args.order}, Dirichlet all faces")
    if args.mesh == "rod":
        return (f"SEM {kind} Jacobi-PCG, {args.iters} iters/step; 17x17-pin rod bundle, 27744 curved elements per "
                f"layer, {args.rod_layers} layers per GPU ({args.rod_layers * world} total, z-slabs), N={args.order}, "
                + ("Dirichlet on pins, walls, inlet" if args.h2 != 0.0 else "Dirichlet on the outlet plane"))
    return (f"SEM {kind} Jacobi-PCG, {args.iters} iters/step; {EX}x{EY}x{args.ez} elements per GPU "
            f"(box {EX}x{EY}x{args.ez * world} elements on [0,1]x[0,1]x[0,{args.ez * world / EX:g}], cubic elements, "
            f"z-slabs), N={args.order}, bubble-deformed, Dirichlet all faces")


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append(parts)

    def mark(self):
        """Samples before this call are outside the timed region."""
        self.start_idx = len(self.samples)

    def stop(self):
        self.samples = self.samples[getattr(self, "start_idx", 0):] or self.samples[-3:]
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def pcg_bytes_per_local_point(info, N):
    """Algorithmic HBM bytes per local point of one UNFUSED Jacobi-PCG iteration:
    Ax (u, 6 metric factors, w) + gs (20 B per shared copy + 4 B per run) + the CG vector updates
    (64 B: x, p, r, w in, x, r out...) + the direction update (32 B) -- what a plain code such as the
    oracle moves; the fused GPU path moves 148 B."""
    nl = info["n_local"]
    gs = (20.0 * (info["n_perm"] + info["n_ifc_perm"]) + 4.0 * (info["n_runs"] + info["n_ifc_runs"])) / nl
    return 64.0 + gs + 64.0 + 32.0


def cpu_baseline(mesh, h2, info, budget_s=8.0):
    """The oracle as it stands (plain C, Dot2 inner products) on the host cores: serial and the
    OpenMP build over all cores of os.sched_getaffinity (same arithmetic, bitwise), median of 3
    timings each of a bounded number of PCG iterations on the N=1 workload mesh; with the host's
    STREAM triad (1 thread / all threads) so the oracle's own CPU roofline fraction is stated."""
    import oracle
    from workloads import meshgen as mg
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    O = oracle.Oracle.from_mesh(mesh)
    b = mg.smooth_field(mesh, seed=1)
    d = O.dinv(1.0, h2)
    bpp = pcg_bytes_per_local_point(info, mesh.N)
    res = {}
    for omp in (False, True):
        oracle.use_openmp(omp)
        L = oracle.lib()
        t0 = time.perf_counter()
        O.pcg(1.0, h2, b, 0.0, 2, dinv=d)                     # probe: seconds per iteration
        per_it = max((time.perf_counter() - t0) / 3.0, 1e-4)
        iters = int(max(2, min(200, budget_s / 3.0 / per_it)))
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            O.pcg(1.0, h2, b, 0.0, iters, dinv=d)
            ts.append(time.perf_counter() - t0)
        dt = statistics.median(ts)
        threads = L.or_threads()
        triad = L.or_triad_gbps(1 << 26, 3)
        gbps = bpp * mesh.n_local * iters / dt / 1e9
        res["omp" if omp else "serial"] = {
            "value": mesh.n_dof * iters / dt / 1e9, "threads": threads, "iters": iters, "median_s": dt,
            "algorithmic_GBps": gbps, "triad_GBps": triad, "frac_of_triad": gbps / triad if triad else None}
    oracle.use_openmp(False)
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    o = res["omp"]
    return {"value": o["value"], "unit": "GDOF/s", "cores": o["threads"], "kind": "oracle",
            "sample": f"{o['iters']} Jacobi-PCG iterations on the N=1 workload mesh, median of 3, plain C oracle "
                      f"(OpenMP over elements / runs / points, {o['threads']} threads; Dot2 inner products sequential)",
            "serial": res["serial"], "all_cores": res["omp"], "cpu_model": model, "cores_available": cores,
            "bytes_per_local_point_per_iter": bpp,
            "note": "algorithmic_GBps = unfused PCG bytes per local point (SURVEY 8(d)) x points x iterations / time; "
                    "triad = a = b + 3c over 3 x 512 MiB, best of 3, the same build's threads"}


def run_reference(args):
    """The reference arm of this tier: the oracle as it stands, timed on the host cores (OpenMP build,
    all cores of os.sched_getaffinity), on the same workload, metric and unit; each step a bounded
    number of PCG iterations."""
    rank, world, _ = rank_env()
    if rank != 0:
        return 0
    mesh = make_mesh(0, 1, args.ez, args.order, args)
    import oracle
    from workloads import meshgen as mg
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    oracle.use_openmp(True)
    O = oracle.Oracle.from_mesh(mesh)
    b = mg.smooth_field(mesh, seed=1)
    d = O.dinv(1.0, args.h2)
    t0 = time.perf_counter()
    O.pcg(1.0, args.h2, b, 0.0, 2, dinv=d)
    per_it = max((time.perf_counter() - t0) / 3.0, 1e-4)
    it_per_step = int(max(1, min(args.iters, 20.0 / max(args.steps + args.warmup, 1) / per_it)))
    for _ in range(args.warmup):
        O.pcg(1.0, args.h2, b, 0.0, it_per_step, dinv=d)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.pcg(1.0, args.h2, b, 0.0, it_per_step, dinv=d)
    dt = time.perf_counter() - t0
    threads = oracle.lib().or_threads()
    val = mesh.n_dof * it_per_step * args.steps / dt / 1e9
    a2 = argparse.Namespace(**vars(args))
    a2.iters = it_per_step
    sample = (f"{it_per_step} Jacobi-PCG iterations per step (the GPU arm runs {args.iters}) on the N=1 workload "
              f"mesh, plain C oracle, OpenMP {threads} threads")
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": val, "unit": "GDOF/s", "n_gpus": 1,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": {"workload": workload_name(a2, 1), "E": mesh.E,
                                                      "N": mesh.N, "n_dof": mesh.n_dof,
                                                      "pcg_iters_per_step": it_per_step},
                      "cpu_baseline": {"value": val, "unit": "GDOF/s", "cores": threads, "kind": "oracle",
                                       "sample": sample},
                      "e2e": {"value": val, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
    return 0


def roofline_of(nek, ctx, info, h2, dev, flush, reps=10, pcg_iters=20):
    """nek_ax (Ax + gs) and the per-kernel classes of a timed PCG pass on one context, against the
    measured copy peak: algorithmic bytes per SURVEY 8(d) (Ax u + 6 factors + w [+ wJ]; gs 20 B per shared
    copy + 4 B per run; the fused PCG Ax adds p, r, Dinv, x in and p, x out)."""
    import torch
    from workloads import meshgen as mg
    stream = torch.cuda.current_stream(dev)
    nl = info["n_local"]
    gs_bytes = 20.0 * info["n_perm"] + 4.0 * info["n_runs"]
    ax_bytes = 8.0 * (8 + (1 if h2 != 0.0 else 0)) * nl
    u = torch.from_numpy(np.random.default_rng(2).standard_normal(nl)).to(dev)
    w = torch.empty_like(u)
    for _ in range(3):
        nek.ax(ctx, 1.0, h2, u, w)
    torch.cuda.synchronize()
    ms = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nek.ax(ctx, 1.0, h2, u, w)
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
    ms /= reps
    out = {"ax_gs": {"ms_per_apply": ms, "gdof_per_s": info["n_dof"] / (ms * 1e-3) / 1e9,
                     "algorithmic_bytes": ax_bytes + gs_bytes, "bytes_per_local_point": (ax_bytes + gs_bytes) / nl,
                     "achieved_GBps": (ax_bytes + gs_bytes) / (ms * 1e-3) / 1e9}}
    nek.get_stats(ctx, reset=True)
    nek.set_timing(ctx, True)
    b = torch.from_numpy(np.random.default_rng(3).standard_normal(nl)).to(dev)
    x = torch.zeros_like(b)
    nek.pcg_solve(ctx, 1.0, h2, b, x, 0.0, pcg_iters)      # capture the timing graph
    nek.get_stats(ctx, reset=True)
    torch.cuda.synchronize()
    nek.pcg_solve(ctx, 1.0, h2, b, x, 0.0, pcg_iters)
    st = nek.get_stats(ctx, reset=True)
    nek.set_timing(ctx, False)
    if st["ax_launches"] and st["ax_ms"] > 0:
        per = st["ax_ms"] / st["ax_launches"]
        byt = st["ax_bytes"] / st["ax_launches"]
        out["pcg_ax"] = {"avg_launch_ms": per, "algorithmic_bytes_per_launch": byt,
                         "achieved_GBps": byt / (per * 1e-3) / 1e9}
    if st["gs_launches"] and st["gs_ms"] > 0:
        per = st["gs_ms"] / st["gs_launches"]
        out["gs"] = {"avg_launch_ms": per, "algorithmic_bytes_per_launch": gs_bytes,
                     "achieved_GBps": gs_bytes / (per * 1e-3) / 1e9}
    if st["vec_launches"] and st["vec_ms"] > 0:
        it = max(1, pcg_iters)
        out["vec_per_iter"] = {"ms": st["vec_ms"] / it, "algorithmic_bytes": 32.0 * nl,
                               "achieved_GBps": 32.0 * nl / (st["vec_ms"] / it * 1e-3) / 1e9,
                               "note": "residual update (w, r, Dinv in; r out) plus the bookkeeping kernels"}
    return out


def with_frac(d, peak):
    for v in d.values():
        if isinstance(v, dict) and "achieved_GBps" in v:
            v["frac"] = v["achieved_GBps"] / peak
    return d


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    rank, world, local = rank_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torch.distributed.run")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2409_19119_b200 import nek
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        comm = nek.comm_from_torch(dev)
    else:
        dist = None
        comm = None

    def barrier():
        if dist:
            dist.barrier()

    def log(msg):
        if os.environ.get("NEK_BENCH_VERBOSE"):
            print(f"[rank {rank}] {msg}", file=sys.stderr, flush=True)

    mesh = make_mesh(rank, world, args.ez, args.order, args)
    log("setup")
    t_setup = time.perf_counter()
    ctx = nek.setup(mesh.E, mesh.N, mesh.xyz, mesh.gid, mesh.mask, comm=comm, device=local)
    t_setup = time.perf_counter() - t_setup
    info = nek.get_info(ctx)
    if args.variant:
        nek.set_variant(ctx, args.variant)
    from workloads import meshgen as mg
    b = torch.from_numpy(mg.smooth_field(mesh, seed=1)).to(dev)
    x = torch.zeros_like(b)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    timing = not args.graph     # a second, per-kernel-timed pass after the timed region
    nek.set_timing(ctx, False)

    clk = ClockSampler(local)
    clk.start()
    time.sleep(1.0)   # let nvidia-smi start sampling before the timed region
    log(f"transport {info['transport']}; warm-up")
    # warm-up (also builds the Jacobi diagonal and, with --graph, the CUDA graph)
    for _ in range(args.warmup):
        nek.pcg_solve(ctx, 1.0, args.h2, b, x, 0.0, args.iters)
    torch.cuda.synchronize()
    nek.get_stats(ctx, reset=True)

    # ---- timed region: K PCG solves, each bracketed by events; L2 flushed between
    barrier(); torch.cuda.synchronize()
    clk.mark()
    evs = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st, it, rr, _ = nek.pcg_solve(ctx, 1.0, args.h2, b, x, 0.0, args.iters)
        e1.record(stream)
        evs.append((e0, e1))
        assert it == args.iters, (st, it)
    torch.cuda.synchronize(); barrier()
    clocks = clk.stop()
    t_ms = sum(a.elapsed_time(c) for a, c in evs)
    launch_stats = nek.get_stats(ctx, reset=True)

    # ---- kernel-timing pass: the same solves again with CUDA events around every kernel class
    # (event-record nodes inside the graph); the events cost ~5 us each, so this pass gives the
    # per-kernel durations for the roofline and the timed region above gives `value`.
    stats = launch_stats
    kt_ms = None
    kt_steps = 0
    if timing:
        nek.set_timing(ctx, True)
        nek.pcg_solve(ctx, 1.0, args.h2, b, x, 0.0, args.iters)          # capture the timing graph
        nek.get_stats(ctx, reset=True)
        kt_steps = max(1, min(args.steps, 5))
        barrier(); torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kt_ms = 0.0
        for _ in range(kt_steps):
            flush.fill_(1)
            ev0.record(stream)
            nek.pcg_solve(ctx, 1.0, args.h2, b, x, 0.0, args.iters)
            ev1.record(stream)
            ev1.synchronize()
            kt_ms += ev0.elapsed_time(ev1)
        torch.cuda.synchronize(); barrier()
        stats = nek.get_stats(ctx, reset=True)
        nek.set_timing(ctx, False)

    log("timed PCG done")
    # ---- Ax+gs alone (nek_ax), same flush discipline
    u = torch.from_numpy(mg.smooth_field(mesh, seed=2)).to(dev)
    w = torch.empty_like(u)
    for _ in range(3):
        nek.ax(ctx, 1.0, args.h2, u, w)
    reps = 20
    barrier(); torch.cuda.synchronize()
    ax_ms = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nek.ax(ctx, 1.0, args.h2, u, w)
        e1.record(stream)
        e1.synchronize()
        ax_ms += e0.elapsed_time(e1)
    barrier()
    axstats = nek.get_stats(ctx, reset=True)

    log("ax done")
    # ---- end to end through the public API with pinned host buffers
    bh = torch.empty(mesh.n_local, dtype=torch.float64, pin_memory=True)
    bh.copy_(b.cpu())
    xh = torch.empty(mesh.n_local, dtype=torch.float64, pin_memory=True)
    nek.set_timing(ctx, False)
    nek.pcg_solve(ctx, 1.0, args.h2, bh, xh, 0.0, args.iters)
    e2e_steps = max(1, min(args.steps, 5))
    barrier(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        nek.pcg_solve(ctx, 1.0, args.h2, bh, xh, 0.0, args.iters)
    torch.cuda.synchronize(); barrier()
    e2e_s = (time.perf_counter() - t0) / e2e_steps

    # ---- time to solution, Jacobi-PCG vs pMG-PCG (NEXT #1), outside the headline metric
    pmg = None
    pm = [0.0] * 5
    if not args.no_pmg:
        tol = 1e-8
        nek.pcg_solve(ctx, 1.0, args.h2, b, x, tol, 5000)   # first: sizes the history buffer both graphs use
        P = nek.PMG(ctx, mesh.xyz, 1.0, args.h2)
        P.solve(b, x, tol, 500)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        barrier(); torch.cuda.synchronize()
        evs[0].record(stream)
        _, itj, _, _ = nek.pcg_solve(ctx, 1.0, args.h2, b, x, tol, 5000)
        evs[1].record(stream)
        evs[2].record(stream)
        pst, itp, prr, _ = P.solve(b, x, tol, 500)
        evs[3].record(stream)
        z = torch.empty_like(b)
        evs[4].record(stream)
        P.apply(b, z)
        evs[5].record(stream)
        torch.cuda.synchronize(); barrier()
        pm = [evs[0].elapsed_time(evs[1]), evs[2].elapsed_time(evs[3]), evs[4].elapsed_time(evs[5])]
        pinfo = P.info()
        P.free()
        itp32 = None
        if args.order <= 9:     # FP32 preconditioner (NEXT #3), same schedule
            P32 = nek.PMG(ctx, mesh.xyz, 1.0, args.h2, precision=1)
            P32.solve(b, x, tol, 500)
            barrier(); torch.cuda.synchronize()
            evs[2].record(stream)
            _, itp32, _, _ = P32.solve(b, x, tol, 500)
            evs[3].record(stream)
            evs[4].record(stream)
            P32.apply(b, z)
            evs[5].record(stream)
            torch.cuda.synchronize(); barrier()
            pm += [evs[2].elapsed_time(evs[3]), evs[4].elapsed_time(evs[5])]
            P32.free()
        else:
            pm += [0.0, 0.0]
        pmg = {"tol": tol, "orders": pinfo["orders"], "degree": pinfo["degree"],
               "coarse_degree": pinfo["coarse_degree"], "iters": itp, "jacobi_iters": itj}
    log("pmg done")
    # ---- projection initial guess (NEXT #2) over a drifting right-hand-side sequence
    proj = None
    pj = [0.0] * 2
    if not args.no_pmg:
        b1 = torch.from_numpy(mg.smooth_field(mesh, seed=4)).to(dev)
        its = {}
        for k, L in enumerate((0, 8)):
            Pj = nek.Projection(ctx, L)
            seq = []
            barrier(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for t in range(12):
                bt = b + (0.01 * t) * b1
                _, it, _ = Pj.solve(1.0, args.h2, bt, x, 1e-8, 5000)
                seq.append(it)
            e1.record(stream)
            torch.cuda.synchronize(); barrier()
            pj[k] = e0.elapsed_time(e1)
            its[L] = seq
            Pj.free()
        proj = {"sequence": "b_t = b0 + 0.01 t b1, t = 0..11, Jacobi-PCG to 1e-8 (S:385)",
                "iters_L0": its[0], "iters_L8": its[8]}
    log("projection done")
    # ---- dealiased advection makef (NEXT #4) on the same mesh: CUDA-event time per apply, L2 flushed
    mk = None
    mkv = [0.0]
    if not args.no_pmg and args.order <= 9:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from makef_bench import makef_cost
        K = nek.Makef(ctx, mesh.xyz)
        Uv = [torch.from_numpy(mg.smooth_field(mesh, seed=s)).to(dev) for s in (5, 6, 7)]
        Fv = [torch.empty_like(Uv[0]) for _ in range(3)]
        for _ in range(3):
            K.apply(*Uv, *Fv)
        barrier(); torch.cuda.synchronize()
        tot = 0.0
        for _ in range(5):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); K.apply(*Uv, *Fv); e1.record(stream); e1.synchronize()
            tot += e0.elapsed_time(e1)
        mkv = [tot / 5]
        mb, mf = makef_cost(args.order)
        mk = {"M": K.M, "bytes_per_element": mb, "flops_per_element": mf, "fp64_peak_tflops": nek.probe_fp64_tflops(local)}
        K.free()
        del Uv, Fv
    log("makef done")
    # ---- peaks measured on this box: FP64 streaming HBM, shared memory, FP64 FMA;
    # at N > 1 also NCCL allreduce latency of the PCG scalars and pairwise send/recv bandwidth
    peaks_box = None
    if not args.no_peaks:
        hb = nek.probe_hbm_gbps(local, 4 << 30)
        peaks_box = {"hbm_fp64_GBps": hb, "smem_TBps": nek.probe_smem_tbps(local),
                     "fp64_fma_TFLOPs": nek.probe_fp64_tflops(local),
                     "note": "double2 read / write / copy kernels over 4 GiB (best of 5), conflict-free "
                             "ld.shared.f64, register FMA chains; CUDA events"}
        if dist:
            lat = {}
            for cnt in (1, 2):
                t = torch.zeros(cnt, dtype=torch.float64, device=dev)
                for _ in range(20):
                    dist.all_reduce(t)
                barrier(); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(200):
                    dist.all_reduce(t)
                e1.record(stream); e1.synchronize()
                lat[f"{8 * cnt}B_us"] = e0.elapsed_time(e1) * 1e3 / 200
            bw = {}
            for nb in (1 << 16, 1 << 20, 1 << 26):
                buf = torch.zeros(nb // 8, dtype=torch.float64, device=dev)
                reps = 20
                for _ in range(3):       # warm-up (connection setup on the first transfer)
                    if rank == 0:
                        dist.send(buf, 1)
                    elif rank == 1:
                        dist.recv(buf, 0)
                barrier(); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(reps):
                    if rank == 0:
                        dist.send(buf, 1)
                    elif rank == 1:
                        dist.recv(buf, 0)
                e1.record(stream); e1.synchronize()
                ms = e0.elapsed_time(e1)
                msv = torch.tensor([ms if rank < 2 else 0.0], dtype=torch.float64, device=dev)
                dist.all_reduce(msv, op=dist.ReduceOp.MAX)
                bw[f"{nb >> 10}KiB"] = nb * reps / (float(msv) * 1e-3) / 1e9
            peaks_box["nccl_allreduce_latency"] = lat
            peaks_box["nccl_sendrecv_GBps_rank0_to_1"] = bw
    log("peaks done")
    # ---- beyond-L2 point (N = 1, box workload): 16 x 16 x 128 elements (11.2M DOF, vectors of 134 MB),
    # where neither the vectors nor the metric factors fit in the L2 -- the HBM roofline proper
    beyond = None
    if world == 1 and args.mesh == "box" and not args.no_beyond:
        mb = make_mesh(0, 1, 128, args.order)
        cb = nek.setup(mb.E, mb.N, mb.xyz, mb.gid, mb.mask, device=local)
        ib = nek.get_info(cb)
        peak_b = 6457.1
        try:
            peak_b = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            pass
        beyond = with_frac(roofline_of(nek, cb, ib, args.h2, dev, flush), peak_b)
        beyond["config"] = {"workload": f"{EX}x{EY}x128 elements, N={args.order}, bubble box", "E": mb.E,
                            "n_dof": mb.n_dof, "n_local": mb.n_local, "l2_keep": ib["l2_keep"],
                            "peak_GBps": peak_b}
        nek.free(cb)
        del mb
    log("beyond-L2 done")

    # ---- max over ranks
    vals = torch.tensor([t_ms, ax_ms, e2e_s] + pm + pj + mkv, dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    t_ms, ax_ms, e2e_s = [float(v) for v in vals.cpu()[:3]]
    pm = [float(v) for v in vals.cpu()[3:3 + len(pm)]]
    pj = [float(v) for v in vals.cpu()[3 + len(pm):3 + len(pm) + len(pj)]]
    mkv = [float(v) for v in vals.cpu()[3 + len(pm) + len(pj):]]
    n_dof_total = mesh.n_dof * world
    if mk is not None:
        ms = mkv[0]
        gbs = mk["bytes_per_element"] * mesh.E / (ms * 1e-3) / 1e9
        tfs = mk["flops_per_element"] * mesh.E / (ms * 1e-3) / 1e12
        mk.update({"ms_per_apply": ms, "gdof_per_s": n_dof_total / (ms * 1e-3) / 1e9, "algorithmic_GBps": gbs,
                   "algorithmic_TFLOPs": tfs, "fp64_frac": tfs / mk["fp64_peak_tflops"],
                   "note": "u, v, w in, 9 M^3 lattice factors, 3 outputs per element; flops of the sum-factorised "
                           "algorithm; FP64 peak = nek_probe_dfma_tflops (register FMA chains, measured here)"})
    if proj is not None:
        proj.update({"ms_L0": pj[0], "ms_L8": pj[1], "speedup": pj[0] / pj[1] if pj[1] > 0 else None})
    if pmg is not None:
        pmg.update({"ms": pm[1], "jacobi_ms": pm[0], "speedup": pm[0] / pm[1] if pm[1] > 0 else None,
                    "ms_per_vcycle": pm[2],
                    "fp32": {"iters": itp32, "ms": pm[3], "ms_per_vcycle": pm[4],
                             "speedup_vs_fp64_pmg": pm[1] / pm[3] if pm[3] > 0 else None},
                    "note": "time to ||r|| <= 1e-8 ||b|| on the same mesh and right-hand side, CUDA events, "
                            "max over ranks; pMG schedule / Chebyshev degrees as listed (DESIGN.md readings P1-P7)"})
    value = n_dof_total * args.iters * args.steps / (t_ms * 1e-3) / 1e9
    ax_gdofs = n_dof_total * reps / (ax_ms * 1e-3) / 1e9

    if rank == 0:
        roofline = None
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        peak = peaks.get("hbm_gbs", 6650.0)
        peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
        union = world > 1 and stats.get("axu_spans", 0) > 0 and stats.get("axu_ms", 0) > 0
        if timing and stats["ax_launches"] > 0 and stats["ax_ms"] > 0:
            per_launch_ms = stats["ax_ms"] / stats["ax_launches"]
            per_launch_bytes = stats["ax_bytes"] / stats["ax_launches"]
            if union:   # N > 1: the boundary and interior launches overlap; bytes of both / their union time
                per_launch_ms = stats["axu_ms"] / stats["axu_spans"]
                per_launch_bytes = stats["ax_bytes"] / stats["axu_spans"]
            achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
            traffic = None
            try:
                tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
                traffic = tr.get(f"ax_N{args.order}_E{mesh.E}")
            except Exception:
                pass
            roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": traffic,
                        "kernel": ("ax_v5 (SEM Helmholtz apply, DMMA, fused PCG prologue)" if args.order == 7 else
                                   "ax_v6 (SEM Helmholtz apply, TMA metric ring, fused PCG prologue)"),
                        "peak_source": peak_src, "algorithmic_bytes_per_launch": per_launch_bytes,
                        "avg_launch_ms": per_launch_ms,
                        "share_of_step": stats["ax_ms"] / kt_ms if kt_ms else None,
                        "timing": "CUDA event-record nodes around each kernel in a second pass of the same "
                                  f"workload ({kt_steps} solves) right after the timed region"
                                  + ("; N > 1: per operator, the union time of the concurrent boundary and "
                                     "interior Ax launches (first start to last end) and the bytes of both"
                                     if union else "")}
        nl = mesh.n_local
        gsb = 20.0 * (info["n_perm"] + info["n_ifc_perm"]) + 4.0 * (info["n_runs"] + info["n_ifc_runs"])
        axb = 8.0 * (8 + (1 if args.h2 != 0.0 else 0)) * nl
        ax_gs = {"gdof_per_s": ax_gdofs, "ms_per_apply": ax_ms / reps,
                 "algorithmic_bytes_per_gpu": axb + gsb, "bytes_per_local_point": (axb + gsb) / nl,
                 "achieved_GBps": (axb + gsb) / (ax_ms / reps * 1e-3) / 1e9,
                 "note": "nek_ax = Ax (u, 6 metric factors, w) + local gs (20 B per shared copy + 4 B per run, "
                         "SURVEY 8(d)) [+ halo]; L2 flushed before every apply"}
        ax_gs["frac"] = ax_gs["achieved_GBps"] / peak
        if timing and stats["gs_launches"] > 0 and stats["gs_ms"] > 0:
            per = stats["gs_ms"] / stats["gs_launches"]
            lgs = 20.0 * info["n_perm"] + 4.0 * info["n_runs"]
            ax_gs["gs_kernel"] = {"avg_launch_ms": per, "algorithmic_bytes_per_launch": lgs,
                                  "achieved_GBps": lgs / (per * 1e-3) / 1e9,
                                  "frac": lgs / (per * 1e-3) / 1e9 / peak}
        out = {
            "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong" if args.mesh == "cfg3" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args, world), "E_per_gpu": mesh.E, "N": mesh.N,
                       "n_dof_per_gpu": mesh.n_dof, "n_local_per_gpu": mesh.n_local,
                       "pcg_iters_per_step": args.iters, "h1": 1.0, "h2": args.h2,
                       "l2": "flushed between steps (256 MiB write outside the timed events)",
                       "parallelism": f"dp{world} (element z-slabs; " + {
                           0: "one GPU, no exchange)",
                           1: "NCCL halo send/recv + allgather reductions)",
                           2: "halo and reductions through NVLink peer memory)"}[info["transport"]],
                       "timing": f"CUDA graph of {min(args.iters, 20)} PCG iterations per replay, device time by CUDA events",
                       "l2_resident": {"keep": info["l2_keep"], "setaside_bytes": info["l2_setaside"],
                                       "setaside_max": info["l2_setaside_max"]},
                       "setup_s": t_setup},
            "pcg_iter_per_s": args.iters * args.steps / (t_ms * 1e-3),
            "ax_gs": ax_gs,
            "beyond_l2": beyond,
            "kernel_ms_per_step": ({k: stats[k] / kt_steps for k in ("ax_ms", "gs_ms", "halo_ms", "vec_ms")}
                                   if kt_ms else None),
            "gpu_launches": int(launch_stats["launches"]),
            "e2e": {"value": n_dof_total * args.iters / e2e_s / 1e9, "unit": "GDOF/s",
                    "h2d_bytes_per_step": mesh.n_local * 8, "d2h_bytes_per_step": mesh.n_local * 8},
            "roofline": roofline, "clocks": clocks, "pmg": pmg, "projection": proj, "makef": mk,
            "halo": {"doubles_per_gs": info["halo_doubles"], "neighbors": info["n_neighbors"],
                     "transport": {0: "none", 1: "nccl", 2: "nvlink-p2p"}[info["transport"]],
                     "GBps": (info["halo_doubles"] * 8 * args.iters / (stats["halo_ms"] / kt_steps * 1e-3) / 1e9
                              if kt_ms and stats["halo_ms"] > 0 else None),
                     "ms_per_step": stats["halo_ms"] / kt_steps if kt_ms else None,
                     "note": "rank 0's interface doubles sent per exchange x iterations / event time of its "
                             "halo kernels (pack + peer stores, or NCCL send/recv)"},
            "peaks_box": peaks_box,
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(mesh, args.h2, info)
        print(json.dumps(out), flush=True)
    nek.free(ctx)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
