#!/usr/bin/env python
"""bench.py — velocity DoFs/s per SIPG viscous apply (FP64, k=3/4) on B200: BASELINE.json's metric.

Workload (N=1 and the scaling runs): **C5**, the largest single-GPU configuration of BASELINE.json
and the strong-scaling config of north_star: backward-facing step (h = 1, expansion ratio 2, inlet
80x32x32 + outlet 448x64x32 graded hex cells = 999,424 cells), k = 3 (191,863,808 velocity DoFs),
Carreau nu (nu0 = 1, nu_inf = 1e-4, lambda = 10, n = 0.5) from the seeded u_lin of DESIGN.md §4,
src uniform[-1,1] from seed 0.  One step = one viscous (Picard) apply through the C ABI
(dgvv_apply_viscous).  Each 1.5 GB vector is > 126 MB L2 (no flush needed); two src/dst pairs rotate.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|3|5]
                    [--no-ops] [--no-cpu-baseline]

Roofline: the apply is FP64-bound ("bound": "alu"): achieved = algorithmic flops
per launch (§8(d): 12n + 96 + 10 + 135/n per DoF on Cartesian cells, faces counted once) / the
launch's mean duration, against the MEASURED DFMA peak of profiles/fp64_peak.json.  The HBM side
(algorithmic bytes: src + dst + the stored nu = 16 + (8/3)(1 + 6/n) B/DoF, and the 16 B/DoF floor)
is in "roofline_other"; "traffic" is ncu's DRAM bytes per launch (profiles/r02_ncu_traffic.json).
At N=1 the line also carries "ops": every other §8(d) op (C2 apply, C3 Picard / Newton /
update_viscosity, C4 Poisson apply / Chebyshev(5) / V-cycle), each the median of 5 timed loops,
with its fractions by §8(d)'s counting.

--impl reference times the CPU oracle (oracle/, full-tensor NumPy fp64) on a bounded sample of the
same workload on this host's cores — the tier's reference arm.  Under torchrun (N > 1) every rank
owns an x-slab of the C5 mesh (strong scaling: total work fixed), exchanges ghost data with NCCL
each apply (overlapped with the interior cells) and rank 0 prints one JSON line (max over ranks).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from inputs import bfs, cube, deformed_cube, uniform  # noqa: E402

METRIC = "velocity DoFs/s per SIPG viscous apply (FP64, k=3/4)"

C2_LAW = {"kind": "exp", "rate": np.log(100.0) / 3.0}
C3_LAW = {"kind": "carreau", "eta0": 1.0, "eta_inf": 1e-3, "lam": 1.0, "n": 0.5}
C4_LAW = {"kind": "exp", "rate": -np.log(1.0e4) / 3.0}
C5_LAW = {"kind": "carreau", "eta0": 1.0, "eta_inf": 1e-4, "lam": 10.0, "n": 0.5}

CONFIGS = {
    2: dict(name="C2", mesh=lambda: deformed_cube(32, 3), k=3, law=C2_LAW,
            desc="C2: 32^3 hex deformed (amp 0.05, degree-3 iso-parametric), k=3, nu=exp(ln(1e2)(x+y+z)/3)"),
    3: dict(name="C3", mesh=lambda: cube(64), k=4, law=C3_LAW,
            desc="C3: 64^3 Cartesian hex, k=4, Carreau nu0=1 nu_inf=1e-3 lambda=1 n=0.5 from 8-mode u_lin"),
    5: dict(name="C5", mesh=lambda: bfs(), k=3, law=C5_LAW,
            desc="C5: backward-facing step, 999,424 graded hex, k=3 (191.9M DoFs), Carreau nu0=1 nu_inf=1e-4 "
                 "lambda=10 n=0.5 from Poiseuille + 8-mode u_lin"),
}


# ---------------------------------------------------------------------- peaks and §8(d) counting
def load_peaks():
    """HBM: MEASURED_PEAKS.json (driver-written copy bandwidth); FP64: profiles/fp64_peak.json
    (scripts/fp64_peak.cu, DFMA, sustained); fallbacks are the guide's nominal figures."""
    hbm, hsrc = 7700.0, "fallback (B200_PROFILING.md nominal)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        hbm, hsrc = json.load(open(p))["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)"
    fp64, fsrc = 148 * 64 * 2 * 1.965e9 / 1e12, "nominal (148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz)"
    q = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(q):
        fp64 = json.load(open(q))["fp64_dfma_tflops_sustained"]
        fsrc = "measured (profiles/fp64_peak.json: DFMA microbenchmark, sustained)"
    return hbm, hsrc, fp64, fsrc


FP64_NOMINAL = 148 * 64 * 2 * 1.965e9 / 1e12


def visc_flops_per_dof(n, general):
    """sum factorisation, collocation basis, each face once."""
    return (12 * n + 96 + 40 + 315 / n) if general else (12 * n + 96 + 10 + 135 / n)


def visc_bytes_per_dof(n):
    """src + dst (16 B/DoF) + the stored nu at cell and own face points."""
    return 16.0 + (8.0 / 3.0) * (1.0 + 6.0 / n)


def fracs(ms, flops, bytes_, hbm, fp64):
    t = ms * 1e-3
    d = {"ms": ms}
    if flops is not None:
        d["alg_gflop"] = flops / 1e9
        d["fp64_tflops"] = flops / t / 1e12
        d["fp64_frac"] = flops / t / 1e12 / fp64
    if bytes_ is not None:
        d["alg_gb"] = bytes_ / 1e9
        d["hbm_gbs"] = bytes_ / t / 1e9
        d["hbm_frac"] = bytes_ / t / 1e9 / hbm
    return d


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x1: "gpu_idle", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev_index=0, period=0.001):
        self.samples, self.reasons = [], set()
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def result(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------- CPU oracle (reference arm)
def _ulin(cfg, m, k):
    from inputs.vectors import c3_linearization, c5_linearization
    return (c3_linearization if cfg["name"] == "C3" else c5_linearization)(m, k)


def time_cpu_oracle(cfg, seconds=15.0, max_cells=4096, mesh=None, ulin=None):
    """The oracle as it stands (never tuned) on a bounded random sample of the workload's cells."""
    from oracle import dg
    m = mesh if mesh is not None else cfg["mesh"]()
    k = cfg["k"]
    d = dg.Disc(m, k)
    u = uniform(0, m.n_cells * 3 * d.N)
    law = cfg["law"]
    if law["kind"] == "carreau":
        nu = dg.CarreauNu(d, ulin if ulin is not None else _ulin(cfg, m, k), law)
    else:
        nu = dg.AnalyticNu(d, law)
    rng = np.random.default_rng(11)
    c0 = np.sort(rng.choice(m.n_cells, 32, replace=False))          # calibrate, then size the sample
    t = time.perf_counter()
    dg.viscous_apply(d, u, nu, cells=c0)
    rate = 32 / (time.perf_counter() - t)
    ncell = int(max(32, min(max_cells, rate * seconds)))
    cells = np.sort(rng.choice(m.n_cells, ncell, replace=False))
    t = time.perf_counter()
    dg.viscous_apply(d, u, nu, cells=cells)
    dt = time.perf_counter() - t
    dofs = ncell * 3 * d.N
    cores = len(os.sched_getaffinity(0))
    return {"value": dofs / dt, "unit": "DoFs/s", "cores": cores, "kind": "oracle",
            "sample": f"oracle viscous apply on {ncell} of {m.n_cells} {cfg['name']} cells "
                      f"({dofs} DoFs, {dt:.1f} s, full-tensor NumPy fp64)", "seconds": dt, "dofs": dofs}


def run_reference(args, rank, world):
    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    m = cfg["mesh"]()
    ulin = _ulin(cfg, m, cfg["k"]) if cfg["law"]["kind"] == "carreau" else None
    per = max(2.0, 60.0 / max(1, args.steps))
    steps = [time_cpu_oracle(cfg, seconds=per, max_cells=1024, mesh=m, ulin=ulin) for _ in range(args.steps)]
    tot_dofs = sum(s["dofs"] for s in steps)
    tot_t = sum(s["seconds"] for s in steps)
    v = tot_dofs / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "DoFs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "dofs": None},
            "cpu_baseline": {"value": v, "unit": "DoFs/s", "kind": "oracle", "cores": steps[0]["cores"],
                             "sample": steps[0]["sample"]},
            "e2e": {"value": v, "unit": "DoFs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- GPU arm
def _nccl_version():
    try:
        import torch
        v = torch.cuda.nccl.version()
        return ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception:
        return None


def _dist_setup(world, rank):
    """torch.distributed (NCCL) for barriers/timing reductions; the library's own NCCL
    communicator for the ghost exchange (unique id broadcast through torch.distributed)."""
    import torch
    import torch.distributed as dist
    from paper_2506_14424_b200.dgvv import nccl_comm_init, nccl_unique_id
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    return nccl_comm_init(bytes(uid.cpu().numpy().tobytes()), world, rank)


def median_loop_ms(fn, n_calls, reps=5, warm=3):
    """SURVEY §8(d) protocol: 3 warm-up calls, then `reps` loops of n_calls, CUDA events on the
    launching stream, median of the loop times / n_calls."""
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(n_calls):
            fn()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / n_calls)
    return statistics.median(ts)


def run_ops(hbm, fp64):
    """Every other §8(d) op on its config, same process, same counting (B_alg / F_alg from the
    §8(d) formulas and table)."""
    import torch
    from inputs.vectors import c3_linearization
    from paper_2506_14424_b200 import _abi as A
    from paper_2506_14424_b200.dgvv import Context

    def dev(x):
        return torch.from_numpy(np.ascontiguousarray(x)).cuda()

    ops = {}
    # C2: deformed 32^3, k = 3, 100 applies per loop (vectors 50 MB: 4 rotating pairs > L2)
    m = deformed_cube(32, 3)
    ctx = Context(m, 3, visc_law=C2_LAW)
    N = 3 * ctx.n_dofs(0)
    srcs = [dev(uniform(100 + i, N)) for i in range(4)]
    dsts = [torch.empty_like(srcs[0]) for _ in range(4)]
    it = [0]

    def c2():
        i = it[0] = (it[0] + 1) % 4
        ctx.apply_viscous(srcs[i], dsts[i])
    ms = median_loop_ms(c2, 100)
    ops["C2_apply_viscous"] = dict(fracs(ms, N * visc_flops_per_dof(4, True), N * visc_bytes_per_dof(4), hbm, fp64),
                                   dofs=N, gdofs_per_s=N / ms / 1e6)
    del ctx, srcs, dsts
    # C3: 64^3, k = 4, Carreau
    m = cube(64)
    ctx = Context(m, 4, visc_law=C3_LAW)
    N = 3 * ctx.n_dofs(0)
    ul = dev(c3_linearization(m, 4))
    ms = median_loop_ms(lambda: ctx.update_viscosity(ul), 5)
    ops["C3_update_viscosity"] = dict(fracs(ms, N * 155.0, N * 13.9, hbm, fp64), dofs=N,
                                      note="K3 Carreau nu at cell + own face points, incl. one host read of the "
                                           "domain-check flag")
    src = dev(uniform(0, N))
    dst = torch.empty_like(src)
    ms = median_loop_ms(lambda: ctx.apply_viscous(src, dst), 20)
    ops["C3_apply_viscous"] = dict(fracs(ms, N * visc_flops_per_dof(5, False), N * visc_bytes_per_dof(5), hbm, fp64),
                                   dofs=N, gdofs_per_s=N / ms / 1e6)
    ctx.apply_linearized_viscous(src, dst)           # derives the Newton point data once per linearisation
    ms = median_loop_ms(lambda: ctx.apply_linearized_viscous(src, dst), 20)
    ops["C3_apply_linearized_viscous"] = dict(fracs(ms, N * 360.0, N * 24.0, hbm, fp64), dofs=N,
                                              gdofs_per_s=N / ms / 1e6)
    del ctx, ul, src, dst
    # C4: scalar Poisson 64^3, k = 5 -> 3 -> 2 -> 1
    ctx = Context(m, 5, poisson_law=C4_LAW, degrees=[5, 3, 2, 1])
    N = ctx.n_dofs(0)
    b = dev(uniform(0, N))
    x = torch.empty_like(b)
    ms = median_loop_ms(lambda: ctx.apply_poisson(b, x), 20)
    ops["C4_apply_poisson"] = dict(fracs(ms, N * (12 * 6 + 96 + 10 + 120 / 6), N * 16.0, hbm, fp64), dofs=N,
                                   gdofs_per_s=N / ms / 1e6)
    lam = [1.2 * ctx.estimate_lambda_max(A.OP_POISSON, dev(uniform(2, ctx.n_dofs(l))), level=l, steps=20)
           for l in range(4)]
    work = torch.empty(2 * N, dtype=torch.float64, device="cuda")
    ms = median_loop_ms(lambda: ctx.chebyshev_smooth(A.OP_POISSON, x, b, lam[0] / 20, lam[0], 5, True, work), 10)
    ops["C4_chebyshev5_from_zero"] = dict(fracs(ms, 4 * N * 198.0, N * 224.0, hbm, fp64), dofs=N,
                                          bound="hbm (SURVEY §8(d))")
    ms = median_loop_ms(lambda: ctx.vcycle(A.OP_POISSON, b, x, lam), 10)
    ops["C4_vcycle_5_3_2_1"] = dict(fracs(ms, 157e9, 42.3e9, hbm, fp64), dofs=N, bound="hbm (SURVEY §8(d))",
                                    gdofs_per_s=N / ms / 1e6)
    ms = median_loop_ms(lambda: ctx.vcycle_fp32(A.OP_POISSON, b, x, lam), 10)
    ops["C4_vcycle_5_3_2_1_fp32_levels"] = dict(ms=ms, dofs=N, gdofs_per_s=N / ms / 1e6,
                                                note="the paper's single-precision preconditioner levels")
    del ctx
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return ops


def run_ours(args, rank, world):
    import torch
    from paper_2506_14424_b200.dgvv import Context
    from paper_2506_14424_b200.partition import slab_partition

    cfg = CONFIGS[args.config]
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    comm = _dist_setup(world, rank) if world > 1 else None
    mg = cfg["mesh"]()
    k = cfg["k"]
    n = k + 1
    per = 3 * n ** 3
    if world > 1:
        part = slab_partition(mg, world, rank)
        ctx = Context(part, k, visc_law=cfg["law"], n_owned=part.n_owned, n_ghost=part.n_ghost,
                      ghost_global_id=part.ghost_global_id, ghost_owner=part.ghost_owner,
                      first_global_cell=part.first, nccl_comm=comm)
        first, n_own = part.first, part.n_owned
    else:
        ctx = Context(mg, k, visc_law=cfg["law"])
        first, n_own = 0, mg.n_cells
    N_glob = mg.n_cells * per
    N = n_own * per
    general = mg.map_degree > 1
    ulin = None
    if cfg["law"]["kind"] == "carreau":
        ulin = _ulin(cfg, mg, k)
        ctx.update_viscosity(torch.from_numpy(ulin[first * per:(first + n_own) * per].copy()).to(dev))
    src0 = uniform(0, N_glob)[first * per:(first + n_own) * per].copy()
    npairs = 2 if N * 8 > 512e6 else 4
    srcs = [torch.from_numpy(src0 if i == 0 else uniform(100 + i, N)).to(dev) for i in range(npairs)]
    dsts = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(npairs)]
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    W = max(3, args.warmup)
    for i in range(W):
        ctx.apply_viscous(srcs[i % npairs], dsts[i % npairs])
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        barrier()
        start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            ctx.apply_viscous(srcs[i % npairs], dsts[i % npairs])
            ev[i][1].record(stream)
        end.record(stream)
        barrier()
    t_ms = max_over_ranks(start.elapsed_time(end) / args.steps)
    per_launch = [a.elapsed_time(b) for a, b in ev]
    t_med = max_over_ranks(statistics.median(per_launch))
    t_launch = max_over_ranks(sum(per_launch) / len(per_launch))
    value = N_glob / (t_ms * 1e-3)

    # end to end through the public C-ABI call with HOST buffers (pinned): dgvv_apply_viscous_host
    # copies src in and dst out inside the timed region, pipelined with the apply by slabs
    hsrc = torch.from_numpy(src0).pin_memory()
    hdst = torch.empty(N, dtype=torch.float64).pin_memory()
    e_steps = 5 if N * 8 > 512e6 else max(3, min(args.steps, 50))
    for _ in range(2):
        ctx.apply_viscous_host(hsrc, hdst)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e_steps):
        ctx.apply_viscous_host(hsrc, hdst)
    e1.record(stream)
    barrier()
    e_ms = max_over_ranks(e0.elapsed_time(e1) / e_steps)

    hbm, hsrc_, fp64, fsrc = load_peaks()
    # the dominant (only) kernel of a step: one launch per step at N=1 (interior + boundary at N>1);
    # §8(d) algorithmic flops and bytes per launch for the cells this rank owns
    flops = N * visc_flops_per_dof(n, general)
    bytes_alg = N * visc_bytes_per_dof(n)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if os.path.exists(prof) and world == 1:
        traffic = json.load(open(prof)).get(cfg["name"])
    ach = flops / (t_launch * 1e-3) / 1e12
    roof = {"bound": "alu", "achieved": ach, "peak": fp64, "unit": "TFLOP/s", "frac": ach / fp64,
            "traffic": traffic, "peak_source": fsrc, "frac_of_nominal": ach / FP64_NOMINAL,
            "nominal_peak": FP64_NOMINAL, "algorithmic_flops_per_launch": flops,
            "counting": f"SURVEY §8(d): {visc_flops_per_dof(n, general):.2f} flop/DoF "
                        f"({'12n+96+40+315/n' if general else '12n+96+10+135/n'}, n={n}, faces once) x {N} DoFs",
            "launch_ms": t_launch}
    achb = bytes_alg / (t_launch * 1e-3) / 1e9
    other = {"bound": "hbm", "achieved": achb, "peak": hbm, "unit": "GB/s", "frac": achb / hbm,
             "frac_16B_floor": N * 16.0 / (t_launch * 1e-3) / 1e9 / hbm, "peak_source": hsrc_,
             "algorithmic_bytes_per_launch": bytes_alg,
             "counting": f"SURVEY §8(d): src + dst + stored nu = {visc_bytes_per_dof(n):.2f} B/DoF x {N} DoFs"}
    launches = args.steps * (1 if world == 1 else 2 + len(ctx.ghost_layout()))
    exch = None
    if world > 1:                              # per-rank face-trace exchange bytes of one apply
        sent, recv = ctx.exchange_bytes(0)
        t = torch.tensor([float(sent), float(recv)], dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        torch.distributed.all_gather(allt, t)
        exch = {"kind": "face traces (value + d/dxi_n per component and face point), NCCL grouped send/recv on a "
                        "comm stream overlapped with the interior cells",
                "bytes_sent_per_apply": [int(x[0].item()) for x in allt],
                "bytes_received_per_apply": [int(x[1].item()) for x in allt],
                "nccl_version": _nccl_version()}
    line = {"metric": METRIC, "value": value, "unit": "DoFs/s", "n_gpus": world, "steps": args.steps,
            "warmup": W, "ms_per_step": t_ms, "ms_per_step_median": t_med, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "dofs": N_glob, "cells": mg.n_cells, "degree": k,
                       "geometry": "general (iso-parametric)" if general else "cartesian (graded boxes)",
                       "parallelism": (f"x-slab domain decomposition x{world}, NCCL ghost exchange overlapped "
                                       "with the interior cells") if world > 1 else "1 GPU",
                       "l2": f"inputs larger than L2: {npairs} rotating src/dst pairs of {N * 8 / 1e9:.2f} GB",
                       "step": "one dgvv_apply_viscous (Picard operator)"},
            "gpu_launches": launches, "roofline": roof, "roofline_other": other,
            "e2e": {"value": N_glob / (e_ms * 1e-3), "unit": "DoFs/s", "h2d_bytes_per_step": N_glob * 8,
                    "d2h_bytes_per_step": N_glob * 8, "ms_per_step": e_ms,
                    "call": "dgvv_apply_viscous_host (pinned host src/dst, copies inside the timed region)"},
            "clocks": clk.result()}
    if exch is not None:
        line["exchange"] = exch
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = time_cpu_oracle(cfg, seconds=args.cpu_seconds, mesh=mg, ulin=ulin)
        cb.pop("seconds")
        cb.pop("dofs")
        line["cpu_baseline"] = cb
    if world == 1 and not args.no_ops:
        del srcs, dsts, ctx
        torch.cuda.empty_cache()
        line["ops"] = run_ops(hbm, fp64)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        ctx.close()
        from paper_2506_14424_b200 import _abi
        _abi.lib().dgvv_nccl_comm_destroy(comm)
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ops", action="store_true", help="skip the per-op table (C2/C3/C4) at N=1")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
