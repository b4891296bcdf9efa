#!/usr/bin/env python
"""bench.py — velocity DoFs/s per SIPG viscous apply (FP64) on B200, BASELINE.json's metric.

Workload (N=1): BASELINE configs[1] = C2: [0,1]^3, 32^3 hex cells deformed by the sinusoidal
map (amplitude 0.05, degree-3 iso-parametric geometry), k = 3 (6,291,456 velocity DoFs),
nu = exp(ln(100)(x+y+z)/3), src uniform[-1,1] from seed 0.  One step = one viscous apply
through the C ABI (dgvv_apply_viscous).  L2 hygiene: 4 src/dst pairs are rotated (4 x 100 MB
plus ~0.5 GB of streamed metric terms > 126 MB L2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|3|4|5]

--impl reference times the CPU oracle (oracle/, full-tensor quadrature, NumPy fp64) on a
bounded sample of the same workload on this host's cores — the tier's reference arm.
Under torchrun (N > 1) every rank owns a z-slab (x-slab for C5) of the mesh, exchanges ghost
cells with NCCL each apply, and rank 0 prints one JSON line (time = max over ranks).
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

CONFIGS = {
    2: dict(name="C2", mesh=lambda: deformed_cube(32, 3), k=3, law={"kind": "exp", "rate": np.log(100.0) / 3.0},
            desc="C2: 32^3 hex deformed (amp 0.05, degree-3 iso-parametric), k=3, nu=exp(ln(1e2)(x+y+z)/3)"),
    3: dict(name="C3", mesh=lambda: cube(64), k=4,
            law={"kind": "carreau", "eta0": 1.0, "eta_inf": 1e-3, "lam": 1.0, "n": 0.5},
            desc="C3: 64^3 Cartesian hex, k=4, Carreau nu0=1 nu_inf=1e-3 lambda=1 n=0.5 from 8-mode u_lin"),
    5: dict(name="C5", mesh=lambda: bfs(), k=3,
            law={"kind": "carreau", "eta0": 1.0, "eta_inf": 1e-4, "lam": 10.0, "n": 0.5},
            desc="C5: backward-facing step, 999,424 graded hex, k=3, Carreau contrast 1e4"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured", d
    return 6650.0, "fallback", {}


# nominal FP64 (non-tensor) peak: 148 SM x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


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


def algorithmic_bytes_per_cell(n, geo):
    """Bytes one apply must move per cell in this design (each array once): src + dst, the
    neighbour table, and the coefficient data: Cartesian — nu at the cell and own face points
    plus 8 doubles of cell geometry; general geometry — the streamed metric terms J^-1 at cell
    points and own face points, nu*JxW and nu*dA (normals/dA are recomputed), H_K."""
    dof = 3 * n ** 3
    b = 8 * 2 * dof + 4 * 6
    if geo == "general":
        b += 8 * (9 * n ** 3 + n ** 3 + 9 * 6 * n * n + 6 * n * n + 1)
    else:
        b += 8 * (n ** 3 + 6 * n * n + 8)
    return b


# algorithmic flops per vector DoF (collocation basis, faces once)
def algorithmic_flops_per_dof(n, geo):
    return (12 * n + 96 + 40 + 315 / n) if geo == "general" else (12 * n + 96 + 10 + 135 / n)


def time_cpu_oracle(cfg, seconds=15.0, max_cells=4096):
    """The oracle as it stands (never tuned) on a bounded sample of the workload's cells."""
    from oracle import dg
    m = cfg["mesh"]()
    k = cfg["k"]
    d = dg.Disc(m, k)
    u = uniform(0, m.n_cells * 3 * d.N)
    law = cfg["law"]
    if law["kind"] == "carreau":
        from inputs.vectors import c3_linearization, c5_linearization
        ulin = (c3_linearization if cfg["name"] == "C3" else c5_linearization)(m, k)
        nu = dg.CarreauNu(d, ulin, law)
    else:
        nu = dg.AnalyticNu(d, law)
    rng = np.random.default_rng(11)
    # calibrate on a small sample, then size the sample for ~`seconds` of CPU work
    c0 = np.sort(rng.choice(m.n_cells, 64, replace=False))
    t = time.perf_counter()
    dg.viscous_apply(d, u, nu, cells=c0)
    rate = 64 / (time.perf_counter() - t)
    ncell = int(max(64, min(max_cells, rate * seconds)))
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
    steps = []
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state
    per = max(2.0, 60.0 / max(1, args.steps))
    for _ in range(args.steps):
        steps.append(time_cpu_oracle(cfg, seconds=per, max_cells=1024))
    tot_dofs = sum(s["dofs"] for s in steps)
    tot_t = sum(s["seconds"] for s in steps)
    v = tot_dofs / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "DoFs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak" if args.gpus > 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "dofs": None},
            "cpu_baseline": {"value": v, "unit": "DoFs/s", "kind": "oracle", "cores": steps[0]["cores"],
                             "sample": steps[0]["sample"]},
            "e2e": {"value": v, "unit": "DoFs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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


def build_workload(cfg, world, scaling):
    """Global mesh: strong scaling splits the config's mesh; weak scaling (C2) stacks one
    C2 cube per GPU in z so every rank owns exactly the C2 workload."""
    if scaling == "weak" and cfg["name"] == "C2" and world > 1:
        return deformed_cube(32, 3, nz_mult=world)
    return cfg["mesh"]()


def run_ours(args, rank, world):
    import torch
    from paper_2506_14424_b200.dgvv import Context
    from paper_2506_14424_b200.partition import slab_partition

    cfg = CONFIGS[args.config]
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    comm = _dist_setup(world, rank) if world > 1 else None
    scaling = args.scaling or ("weak" if cfg["name"] == "C2" else "strong")
    mg = build_workload(cfg, world, scaling)
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
    geo = "general" if mg.map_degree > 1 else "cartesian"
    if cfg["law"]["kind"] == "carreau":
        from inputs.vectors import c3_linearization, c5_linearization
        ulin = (c3_linearization if cfg["name"] == "C3" else c5_linearization)(mg, k)
        ulin_d = torch.from_numpy(ulin[first * per:(first + n_own) * per].copy()).to(dev)
        ctx.update_viscosity(ulin_d)
    src0 = uniform(0, N_glob)[first * per:(first + n_own) * per].copy()
    npairs = 4
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

    for i in range(max(3, args.warmup)):
        ctx.apply_viscous(srcs[i % npairs], dsts[i % npairs])
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        barrier()
        start.record(stream)
        for i in range(args.steps):
            ctx.apply_viscous(srcs[i % npairs], dsts[i % npairs])
        end.record(stream)
        barrier()
    t_ms = max_over_ranks(start.elapsed_time(end) / args.steps)
    value = N_glob / (t_ms * 1e-3)

    # end to end through the public C-ABI call with HOST buffers (pinned): dgvv_apply_viscous_host
    # copies src in and dst out inside the timed region, pipelined with the apply by slabs
    hsrc = torch.from_numpy(src0).pin_memory()
    hdst = torch.empty(N, dtype=torch.float64).pin_memory()
    e_steps = max(3, min(args.steps, 50))
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

    hbm_peak, peak_src, _ = load_peaks()
    bytes_launch = algorithmic_bytes_per_cell(n, geo) * n_own
    flops_launch = algorithmic_flops_per_dof(n, geo) * N
    t_hbm = bytes_launch / (hbm_peak * 1e9)
    t_alu = flops_launch / (FP64_PEAK_TFLOPS * 1e12)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        traffic = json.load(open(prof)).get(cfg["name"])
    hbm_roof = {"bound": "hbm", "achieved": bytes_launch / (t_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "frac": bytes_launch / (t_ms * 1e-3) / 1e9 / hbm_peak, "traffic": traffic,
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                "algorithmic_bytes_per_launch": bytes_launch}
    alu_roof = {"bound": "alu", "achieved": flops_launch / (t_ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": flops_launch / (t_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                "peak_source": "nominal FP64 148 SM x 64 FMA x 2 x 1.965 GHz (DESIGN.md; measured DFMA 34.2)",
                "algorithmic_flops_per_launch": flops_launch}
    roof, other = (hbm_roof, alu_roof) if t_hbm >= t_alu else (alu_roof, hbm_roof)
    launches = args.steps * (1 if world == 1 else 2 + sum(1 for _ in ctx.ghost_layout()))
    line = {"metric": METRIC, "value": value, "unit": "DoFs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
            "scaling": scaling if world > 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"] + (f"; weak scaling: {world} C2 cubes stacked in z, one per GPU"
                                                  if world > 1 and scaling == "weak" else ""),
                       "dofs": N_glob, "cells": mg.n_cells, "degree": k, "geometry": geo,
                       "parallelism": f"slab domain decomposition x{world}, NCCL ghost-cell exchange" if world > 1 else "1 GPU",
                       "l2": f"{npairs} rotating src/dst pairs ({npairs * 2 * N * 8 / 1e6:.0f} MB) + coefficient/metric "
                             "streams > 126 MB L2", "step": "one dgvv_apply_viscous"},
            "gpu_launches": launches,
            "roofline": roof, "roofline_other": other,
            "e2e": {"value": N_glob / (e_ms * 1e-3), "unit": "DoFs/s", "h2d_bytes_per_step": N_glob * 8,
                    "d2h_bytes_per_step": N_glob * 8, "ms_per_step": e_ms},
            "clocks": clk.result()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = time_cpu_oracle(cfg, seconds=args.cpu_seconds)
        cb.pop("seconds")
        cb.pop("dofs")
        line["cpu_baseline"] = cb
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="multi-GPU: weak (C2 default: one C2 cube per GPU) or strong (split the config's mesh)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
