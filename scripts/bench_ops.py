#!/usr/bin/env python
"""Per-operation B200 timings for every SURVEY §8(a) row on the BASELINE configs (C2-C5).

    python scripts/bench_ops.py [--configs 2,3,4,5] [--reps 5] > profiles/rNN_ops.json

One JSON object per (config, op): median over `reps` loops of N calls (SURVEY §8(d) protocol:
3 warm-up calls, CUDA events on the launching stream), ms per call, DoFs/s, and the
algorithmic-byte / algorithmic-flop fractions of the measured peaks (HBM from
MEASURED_PEAKS.json, FP64 from scripts/fp64_peak.cu, 34.2 TFLOP/s).  Inputs are the seeded
synthetic inputs of DESIGN.md §4.  Not a bench.py line: the driver's metric is bench.py's.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import bfs, cube, deformed_cube, uniform  # noqa: E402
from inputs.vectors import c3_linearization, c5_linearization  # noqa: E402
from paper_2506_14424_b200 import _abi as A  # noqa: E402
from paper_2506_14424_b200.dgvv import Context  # noqa: E402

FP64_MEASURED = 34.2e12
C2_LAW = {"kind": "exp", "rate": np.log(100.0) / 3.0}
C4_LAW = {"kind": "exp", "rate": -np.log(1.0e4) / 3.0}
C3_LAW = {"kind": "carreau", "eta0": 1.0, "eta_inf": 1.0e-3, "lam": 1.0, "n": 0.5}
C5_LAW = {"kind": "carreau", "eta0": 1.0, "eta_inf": 1.0e-4, "lam": 10.0, "n": 0.5}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] * 1e9 if os.path.exists(p) else 6.65e12


def timeit(fn, n_calls, reps):
    for _ in range(3):
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


def report(cfg, op, ms, dofs, bytes_=None, flops=None, note=""):
    d = {"config": cfg, "op": op, "ms": round(ms, 5), "dofs": dofs, "gdofs_per_s": round(dofs / ms / 1e6, 3)}
    if bytes_ is not None:
        d["alg_bytes"] = bytes_
        d["hbm_frac"] = round(bytes_ / (ms * 1e-3) / hbm_peak(), 4)
    if flops is not None:
        d["alg_flops"] = flops
        d["fp64_frac_measured"] = round(flops / (ms * 1e-3) / FP64_MEASURED, 4)
    if note:
        d["note"] = note
    print(json.dumps(d), flush=True)


def visc_bytes(cells, n, general):
    b = 8 * 2 * 3 * n ** 3 + 24
    b += 8 * (10 * n ** 3 + 60 * n * n + 1) if general else 8 * (n ** 3 + 6 * n * n + 8)
    return b * cells


def visc_flops(dofs, n, general):
    return dofs * ((12 * n + 96 + 40 + 315 / n) if general else (12 * n + 96 + 10 + 135 / n))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_c2(reps):
    m = deformed_cube(32, 3)
    ctx = Context(m, 3, visc_law=C2_LAW)
    N = ctx.n_dofs() * 3
    src = [dev(uniform(100 + i, N)) for i in range(4)]
    dst = [torch.empty_like(src[0]) for _ in range(4)]
    it = iter(range(10 ** 9))
    ms = timeit(lambda: ctx.apply_viscous(src[next(it) % 4], dst[0]), 100, reps)
    report("C2", "apply_viscous", ms, N, visc_bytes(m.n_cells, 4, True), visc_flops(N, 4, True))
    # the C2 (deformed, iso-parametric) geometry with C3's Carreau law: Picard and Newton applies
    # of the general-geometry kernels (VERDICT r1 "Hygiene": the general-geometry Newton is the
    # v1 kernel that recomputes nu'(gamma) per point; Cartesian meshes use v3 with stored point data)
    cc = Context(m, 3, visc_law=C3_LAW)
    cc.update_viscosity(dev(c3_linearization(cube(32), 3)))   # the field at the undeformed positions
    ms = timeit(lambda: cc.apply_viscous(src[0], dst[0]), 50, reps)
    report("C2-Carreau", "apply_viscous", ms, N, visc_bytes(m.n_cells, 4, True), visc_flops(N, 4, True))
    ms = timeit(lambda: cc.apply_linearized_viscous(src[0], dst[0]), 50, reps)
    report("C2-Carreau", "apply_linearized_viscous", ms, N, None, None,
           "general-geometry Newton (v1: recomputes the Carreau derivative at every point)")


def run_c3(reps):
    m = cube(64)
    ctx = Context(m, 4, visc_law=C3_LAW)
    N = ctx.n_dofs() * 3
    ulin = dev(c3_linearization(m, 4))
    ms = timeit(lambda: ctx.update_viscosity(ulin), 10, reps)
    cells = m.n_cells
    report("C3", "update_viscosity", ms, N, 8 * cells * (3 * 125 + 125 + 6 * 25), None,
           "K3 Carreau nu at cell + own face points")
    src = dev(uniform(0, N))
    dst = torch.empty_like(src)
    ms = timeit(lambda: ctx.apply_viscous(src, dst), 20, reps)
    report("C3", "apply_viscous", ms, N, visc_bytes(cells, 5, False), visc_flops(N, 5, False))
    ms = timeit(lambda: ctx.apply_linearized_viscous(src, dst), 20, reps)
    report("C3", "apply_linearized_viscous", ms, N, 8 * 3 * N + 8 * 8 * cells, 360.0 * N)


def run_c4(reps):
    m = cube(64)
    degs = [5, 3, 2, 1]
    ctx = Context(m, 5, poisson_law=C4_LAW, degrees=degs)
    N = ctx.n_dofs(0)
    n = 6
    b = dev(uniform(0, N))
    x = torch.empty_like(b)
    cells = m.n_cells
    pb = 8 * cells * (2 * n ** 3 + n ** 3 + 6 * n * n + 8) + 24 * cells
    ms = timeit(lambda: ctx.apply_poisson(b, x), 20, reps)
    report("C4", "apply_poisson_k5", ms, N, pb, N * (12 * n + 96 + 10 + 120 / n))
    dinv = torch.empty_like(b)
    ctx.inverse_diagonal(A.OP_POISSON, dinv)           # first call: module load + K5 kernel
    ctx.set_mass(A.OP_POISSON, 1e-300)                 # two coefficient changes invalidate the cached
    ctx.set_mass(A.OP_POISSON, 0.0)                    # D^-1: the next call runs K5 again (same operator)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.inverse_diagonal(A.OP_POISSON, dinv)
    e1.record()
    e1.synchronize()
    report("C4", "inverse_diagonal_k5_kernel", e0.elapsed_time(e1), N, 8 * cells * (2 * n ** 3 + 12 * n * n) + 24 * cells,
           None, "K5 kernel recomputing the cached D^-1 in place, single shot")
    ms = timeit(lambda: ctx.inverse_diagonal(A.OP_POISSON, dinv), 10, reps)
    report("C4", "inverse_diagonal_k5_cached", ms, N, 8 * 2 * N, None, "later calls copy the cached D^-1")
    lam = []
    for lvl in range(len(degs)):
        v0 = dev(uniform(2, ctx.n_dofs(lvl)))
        lam.append(1.2 * ctx.estimate_lambda_max(A.OP_POISSON, v0, level=lvl, steps=20))
    work = torch.empty(2 * N, dtype=torch.float64, device="cuda")
    ms = timeit(lambda: ctx.chebyshev_smooth(A.OP_POISSON, x, b, lam[0] / 20, lam[0], 5, True, work), 10, reps)
    report("C4", "chebyshev5_from_zero_k5", ms, N, 4 * pb + 8 * N * (2 + 6 * 4), None,
           "4 applies with fused Chebyshev epilogue (x0 = 0)")
    x0 = dev(uniform(3, N))
    xs = x0.clone()
    ms = timeit(lambda: (xs.copy_(x0), ctx.chebyshev_smooth(A.OP_POISSON, xs, b, lam[0] / 20, lam[0], 5, False, work)),
                10, reps)
    report("C4", "chebyshev5_from_x0_k5", ms, N, 5 * pb + 8 * N * (2 + 6 * 5), None, "includes one vector copy")
    ms = timeit(lambda: ctx.vcycle(A.OP_POISSON, b, x, lam), 10, reps)
    report("C4", "vcycle_5_3_2_1", ms, N, None, None, "fine-level DoFs per V-cycle second")
    ms = timeit(lambda: ctx.vcycle_fp32(A.OP_POISSON, b, x, lam), 10, reps)
    report("C4", "vcycle_5_3_2_1_fp32", ms, N, None, None, "every level in FP32 (f1); FP64 b/x converted")
    c = torch.empty(ctx.n_dofs(1), dtype=torch.float64, device="cuda")
    ms = timeit(lambda: ctx.restrict(A.OP_POISSON, 0, b, c), 20, reps)
    report("C4", "restrict_5_to_3", ms, N, 8 * cells * (216 + 64))
    ms = timeit(lambda: ctx.prolongate(A.OP_POISSON, 0, c, x, 1.0), 20, reps)
    report("C4", "prolongate_add_3_to_5", ms, N, 8 * cells * (64 + 2 * 216))


def run_f1(reps):
    """f1: Helmholtz viscous step (mass = 1e3) on C3, PCG to rtol 1e-8, FP64 vs FP32 V-cycle."""
    m = cube(64)
    degs = [4, 2, 1]
    ctx = Context(m, 4, visc_law=C3_LAW, degrees=degs)
    ctx.set_mass(A.OP_VISCOUS, 1.0e3)
    ctx.update_viscosity(dev(c3_linearization(m, 4)))
    lams = [1.2 * ctx.estimate_lambda_max(A.OP_VISCOUS, dev(uniform(2, 3 * ctx.n_dofs(l))), level=l, steps=20)
            for l in range(len(degs))]
    N = 3 * ctx.n_dofs(0)
    b = dev(uniform(0, N))
    for pc in ("vcycle", "vcycle_fp32", "jacobi"):
        x = torch.zeros(N, dtype=torch.float64, device="cuda")
        ctx.cg_solve(A.OP_VISCOUS, b, x, rtol=1e-8, maxit=400, precond=pc, lam_hi_per_level=lams)   # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x.zero_()
        e0.record()
        it, rr = ctx.cg_solve(A.OP_VISCOUS, b, x, rtol=1e-8, maxit=400, precond=pc, lam_hi_per_level=lams)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        report("C3+f1", f"helmholtz_pcg_{pc}", ms, N, None, None,
               f"{it} iterations to rtol 1e-8 (relres {rr:.2e}); {ms / max(it, 1):.3f} ms/iteration")
        x2 = torch.zeros(N, dtype=torch.float64, device="cuda")
        if pc != "jacobi":
            r = dev(uniform(5, N))
            f = ctx.vcycle if pc == "vcycle" else ctx.vcycle_fp32
            ms = timeit(lambda: f(A.OP_VISCOUS, r, x2, lams), 5, reps)
            report("C3+f1", f"viscous_{pc}_4_2_1", ms, N, None, None, "one V-cycle of the Helmholtz operator")


def run_f2(reps):
    """f2: penalty-step operator on the C2 mesh (32^3 deformed, k=3) and on C3's 64^3 k=4 mesh,
    tau ~ |u| h dt (Fehn2018b-sized, P1), apply + Jacobi-PCG to rtol 1e-10."""
    # dt scales both penalty parameters (tau_D dt, tau_C dt): 1e-3 is a CFL-sized step (the operator
    # stays close to the mass matrix, Jacobi suffices), 1e-1 the large steps of the paper's
    # steady cavity runs, where "a multigrid preconditioner is necessary"
    for name, m, k, dt in (("C2", deformed_cube(32, 3), 3, 1e-3), ("C3", cube(64), 4, 1e-3),
                           ("C3 dt=1e-1", cube(64), 4, 1e-1)):
        ctx = Context(m, k, visc_law=C2_LAW)
        rng = np.random.default_rng(11)
        h = 1.0 / round(m.n_cells ** (1 / 3))
        speed = rng.uniform(0.1, 2.0, m.n_cells)
        ctx.set_penalty_parameters(speed * h * dt, speed * dt)
        N = 3 * ctx.n_dofs(0)
        src = dev(uniform(0, N))
        dst = torch.empty_like(src)
        n = k + 1
        general = m.map_degree > 1
        byt = m.n_cells * 8 * (2 * 3 * n ** 3 + 2 + (10 * n ** 3 + 6 * 4 * n * n if general else 8))
        ms = timeit(lambda: ctx.apply_penalty(src, dst), 20, reps)
        report(name + "+f2", "apply_penalty", ms, N, byt, None, "mass + div-div + continuity penalty")
        x = torch.zeros_like(src)
        ctx.cg_solve(A.OP_PENALTY, src, x, rtol=1e-10, maxit=2000, precond="jacobi")
        x.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        it, rr = ctx.cg_solve(A.OP_PENALTY, src, x, rtol=1e-10, maxit=2000, precond="jacobi")
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        report(name + "+f2", "penalty_pcg_jacobi", ms, N, None, None,
               f"{it} iterations to rtol 1e-10 (relres {rr:.2e}); {ms / max(it, 1):.3f} ms/iteration")
        # f2 multigrid: V-cycle-PCG over the p-levels k -> 2 -> 1
        degs = [k, 2, 1]
        cm = Context(m, k, visc_law=C2_LAW, degrees=degs)
        cm.set_penalty_parameters(speed * h * dt, speed * dt)
        t_l, lams = _timed(lambda: [1.2 * cm.estimate_lambda_max(A.OP_PENALTY, dev(uniform(2, 3 * cm.n_dofs(l))),
                                                                 level=l, steps=20) for l in range(3)])
        x = torch.zeros_like(src)
        cm.cg_solve(A.OP_PENALTY, src, x, rtol=1e-10, maxit=2000, precond="vcycle", lam_hi_per_level=lams)
        x.zero_()
        ms, (it, rr) = _timed(lambda: cm.cg_solve(A.OP_PENALTY, src, x, rtol=1e-10, maxit=2000, precond="vcycle",
                                                  lam_hi_per_level=lams))
        report(name + "+f2", "penalty_pcg_vcycle", ms, N, None, None,
               f"{it} iterations to rtol 1e-10 (relres {rr:.2e}); {ms / max(it, 1):.3f} ms/iteration; "
               f"p-levels {degs}; lambda setup (20 Lanczos steps per level) {t_l:.1f} ms")
        del cm


F4_NU = {"kind": "const", "value": 1.0e-3}      # convection-dominated viscous step (high Re)


def run_f4(reps):
    """f4: upwind convective term on the C2 mesh (32^3 deformed, k=3) and C3's mesh (64^3, k=4)
    with a random transport field w = rng(1); the Oseen-type viscous step mass M + A(nu) + C(w)
    (nu = 1e-3 so that convection matters, mass = 1e3 ~ gamma_0/dt for a CFL-limited dt) and
    GMRES(30) with the FP64 / FP32 V-cycle of the symmetric part to rtol 1e-8 (p-levels only, then
    the cph V-cycle; C3 also with a smooth transport field)."""
    for name, m, k, degs in (("C2", deformed_cube(32, 3), 3, [3, 2, 1]), ("C3", cube(64), 4, [4, 2, 1])):
        ctx = Context(m, k, visc_law=F4_NU, degrees=degs)
        N = 3 * ctx.n_dofs(0)
        src = dev(uniform(0, N))
        ctx.set_transport(dev(uniform(1, N)))
        dst = torch.empty_like(src)
        n = k + 1
        general = m.map_degree > 1
        # src + dst + stored point data of w (JxW J^-1 w: 3 per cell point; min({{w}}.n,0) dA: 6 n^2) + nbr
        byt = m.n_cells * (8 * (2 * 3 * n ** 3 + 3 * n ** 3 + 6 * n * n) + 24)
        ctx.apply_convective(src, dst)                 # derives the point data (once per transport field)
        ms = timeit(lambda: ctx.apply_convective(src, dst), 20, reps)
        report(name + "+f4", "apply_convective", ms, N, byt, None, "upwind convective term C(w) u (stored point data of w)")
        ctx.set_mass(0, 1.0e3)
        ms = timeit(lambda: ctx.apply_oseen(src, dst, 1.0), 20, reps)
        report(name + "+f4", "apply_oseen", ms, N, None, None, "mass M + A(nu) + C(w): one fused kernel")
        lams = [1.2 * ctx.estimate_lambda_max(0, dev(uniform(2, 3 * m.n_cells * (kk + 1) ** 3)), level=l, steps=15)
                for l, kk in enumerate(degs)]
        for pc in ("vcycle", "vcycle_fp32"):
            x = torch.zeros_like(src)
            ctx.gmres_solve(src, x, rtol=1e-8, restart=30, maxit=300, precond=pc, lam_hi_per_level=lams)
            x.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            it, rr = ctx.gmres_solve(src, x, rtol=1e-8, restart=30, maxit=300, precond=pc, lam_hi_per_level=lams)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            report(name + "+f4", "gmres_" + pc, ms, N, None, None,
                   f"{it} iterations to rtol 1e-8 (relres {rr:.2e}); {ms / max(it, 1):.3f} ms/iteration")
        # the cph V-cycle (h-levels down to 4^3 at k = 1, direct solve) of the symmetric part
        from inputs import cube_parent_map
        keep, prev, Nc = [], ctx, round(m.n_cells ** (1 / 3))
        while Nc > 4:
            Nc //= 2
            cm = deformed_cube(Nc, 3) if general else cube(Nc)
            c = Context(cm, 1, visc_law=F4_NU)
            c.set_mass(0, 1.0e3)
            parent, octant = cube_parent_map(2 * Nc)
            prev.set_coarse_context(c, parent, octant)
            keep.append(c)
            prev = c
        keep[-1].setup_coarse_solver(0)
        lams_h = lams + [1.2 * c.estimate_lambda_max(0, dev(uniform(2, 3 * c.n_dofs(0))), level=0, steps=15)
                         for c in keep[:-1]] + [1.0]
        fields = [("random w", None)] + ([("smooth w (8-mode Fourier field)", c3_linearization(m, 4))] if not general else [])
        for wname, wv in fields:
            if wv is not None:
                ctx.set_transport(dev(wv))
            for pc in ("vcycle", "vcycle_fp32"):
                x = torch.zeros_like(src)
                ctx.gmres_solve(src, x, rtol=1e-8, restart=30, maxit=300, precond=pc, lam_hi_per_level=lams_h)
                x.zero_()
                ms, (it, rr) = _timed(lambda: ctx.gmres_solve(src, x, rtol=1e-8, restart=30, maxit=300, precond=pc,
                                                              lam_hi_per_level=lams_h))
                report(name + "+f4", "gmres_cph_" + pc + ("_smooth_w" if wv is not None else ""), ms, N, None, None,
                       f"{wname}, cph V-cycle: {it} iterations (relres {rr:.2e}); {ms / max(it, 1):.3f} ms/iteration")
        del keep


def _timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1), out


def run_f3(reps):
    """f3: cph hierarchy on the C4 Poisson problem (64^3, k = 5 -> 3 -> 2 -> 1, then h-levels 32^3 ... 4^3
    at k = 1, direct solve on 4^3 = 512 DoFs) and on the C3 Helmholtz viscous step (64^3, k = 4 -> 2 -> 1,
    h-levels to 4^3, direct solve on 1536 DoFs; mass 1 and 1e3): PCG to 1e-8 with the p-only vs the
    cph V-cycle."""
    from inputs import cube_parent_map
    for name, op, k0, degs, law, masses in (("C4", A.OP_POISSON, 5, [5, 3, 2, 1], C4_LAW, [0.0]),
                                            ("C3", A.OP_VISCOUS, 4, [4, 2, 1], C2_LAW, [1.0, 1.0e3])):
        kw = {"poisson_law": law} if op == A.OP_POISSON else {"visc_law": law}
        nc = 1 if op == A.OP_POISSON else 3
        for mass in masses:
            fine = Context(cube(64), k0, degrees=degs, **kw)
            fine.set_mass(op, mass)
            lams = [1.2 * fine.estimate_lambda_max(op, dev(uniform(2, nc * fine.n_dofs(l))), level=l, steps=20)
                    for l in range(len(degs))]
            N = nc * fine.n_dofs(0)
            b = dev(uniform(0, N))
            x = torch.zeros_like(b)
            tag = f"{name}+f3" + (f" mass={mass:g}" if op == A.OP_VISCOUS else "")
            fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle", lam_hi_per_level=lams)
            x.zero_()
            ms, (it, rr) = _timed(lambda: fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle",
                                                        lam_hi_per_level=lams))
            report(tag, "pcg_vcycle_p_only", ms, N, None, None, f"{it} iterations (relres {rr:.1e}); {ms / max(it, 1):.2f} ms/it")
            ms = timeit(lambda: fine.vcycle(op, b, x, lams), 5, reps)
            report(tag, "vcycle_p_only", ms, N, None, None, "coarsest: Chebyshev(5) on 64^3 k=1")
            prev, Nc, keep = fine, 64, []
            while Nc > 4:
                Nc //= 2
                c = Context(cube(Nc), 1, **kw)
                c.set_mass(op, mass)
                parent, octant = cube_parent_map(2 * Nc)
                prev.set_coarse_context(c, parent, octant)
                keep.append(c)
                if Nc > 4:
                    lams.append(1.2 * c.estimate_lambda_max(op, dev(uniform(2, nc * c.n_dofs(0))), level=0, steps=20))
                prev = c
            ms_setup, nd = _timed(lambda: keep[-1].setup_coarse_solver(op))
            lams.append(1.0)
            report(tag, "setup_coarse_solver", ms_setup, nd, None, None, f"assemble + Gauss-Jordan inverse of {nd} DoFs")
            x.zero_()
            fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle", lam_hi_per_level=lams)
            x.zero_()
            ms, (it, rr) = _timed(lambda: fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle",
                                                        lam_hi_per_level=lams))
            report(tag, "pcg_vcycle_cph", ms, N, None, None, f"{it} iterations (relres {rr:.1e}); {ms / max(it, 1):.2f} ms/it")
            ms = timeit(lambda: fine.vcycle(op, b, x, lams), 5, reps)
            report(tag, "vcycle_cph", ms, N, None, None, f"{fine.chain_levels()} levels, direct solve on 4^3 k=1")
            x.zero_()
            fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle_fp32", lam_hi_per_level=lams)
            x.zero_()
            ms, (it, rr) = _timed(lambda: fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle_fp32",
                                                        lam_hi_per_level=lams))
            report(tag, "pcg_vcycle_cph_fp32", ms, N, None, None,
                   f"{it} iterations (relres {rr:.1e}); {ms / max(it, 1):.2f} ms/it; FP32 levels, FP64 direct solve")
            # c-level: DG p-levels -> continuous Q1 on 64^3 -> Q1 h-levels -> direct on 4^3 (125 vertices)
            ctxs = [fine] + keep
            for c in ctxs:
                c.set_continuous_level()
            lams_c = lams[:len(degs)]
            for c in ctxs[:-1]:
                lams_c.append(1.2 * c.estimate_lambda_max_continuous(op, dev(uniform(2, nc * c.n_vertices)), steps=20))
            ms_setup, nd = _timed(lambda: keep[-1].setup_coarse_solver(op))
            lams_c.append(1.0)
            report(tag, "setup_coarse_solver_continuous", ms_setup, nd, None, None, f"{nd} continuous DoFs")
            x.zero_()
            fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle", lam_hi_per_level=lams_c)
            x.zero_()
            ms, (it, rr) = _timed(lambda: fine.cg_solve(op, b, x, rtol=1e-8, maxit=400, precond="vcycle",
                                                        lam_hi_per_level=lams_c))
            report(tag, "pcg_vcycle_cph_c_level", ms, N, None, None,
                   f"{it} iterations (relres {rr:.1e}); {ms / max(it, 1):.2f} ms/it; DG p -> c (Q1) -> Q1 h -> direct")
            ms = timeit(lambda: fine.vcycle(op, b, x, lams_c), 5, reps)
            report(tag, "vcycle_cph_c_level", ms, N, None, None, f"{fine.chain_levels()} levels")
            del keep, fine, ctxs
            torch.cuda.empty_cache()


def run_step(reps):
    """One Picard-linearised viscous step of the paper's projection scheme on C3's mesh, end to end
    on the GPU: update_viscosity(u_lin) (Carreau nu on every level), inverse diagonals and
    lambda_max (15 Lanczos steps) of every level, then PCG to 1e-8 on gamma_0/dt M + A(nu) with the
    FP32 cph V-cycle (p 4 -> 2 -> 1, h-levels 32^3 ... 4^3 at k = 1, direct solve on 4^3); the
    h-levels carry the analytic C2 law (the Carreau u_lin lives on the fine mesh only).  Each phase
    timed with CUDA events; the step = their sum."""
    from inputs import cube_parent_map
    m = cube(64)
    degs = [4, 2, 1]
    fine = Context(m, 4, visc_law=C3_LAW, degrees=degs)
    fine.set_mass(A.OP_VISCOUS, 1.0e3)
    ulin = dev(c3_linearization(m, 4))
    N = 3 * fine.n_dofs(0)
    keep, prev, Nc = [], fine, 64
    while Nc > 4:
        Nc //= 2
        c = Context(cube(Nc), 1, visc_law=C2_LAW)
        c.set_mass(A.OP_VISCOUS, 1.0e3)
        parent, octant = cube_parent_map(2 * Nc)
        prev.set_coarse_context(c, parent, octant)
        keep.append(c)
        prev = c
    keep[-1].setup_coarse_solver(A.OP_VISCOUS)
    lam_h = [1.2 * c.estimate_lambda_max(A.OP_VISCOUS, dev(uniform(2, 3 * c.n_dofs(0))), level=0, steps=15)
             for c in keep[:-1]]
    b = dev(uniform(0, N))
    x = torch.zeros_like(b)
    v0 = [dev(uniform(2, 3 * fine.n_dofs(l))) for l in range(len(degs))]

    def step():
        t = {}
        def ev():
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            return e
        e0 = ev()
        fine.update_viscosity(ulin)
        e1 = ev()
        lams = [1.2 * fine.estimate_lambda_max(A.OP_VISCOUS, v0[l], level=l, steps=15) for l in range(len(degs))]
        e2 = ev()
        x.zero_()
        it, rr = fine.cg_solve(A.OP_VISCOUS, b, x, rtol=1e-8, maxit=200, precond="vcycle_fp32",
                               lam_hi_per_level=lams + lam_h + [1.0])
        e3 = ev()
        e3.synchronize()
        t["update_viscosity"] = e0.elapsed_time(e1)
        t["diagonals+lambda"] = e1.elapsed_time(e2)
        t["pcg"] = e2.elapsed_time(e3)
        return t, it, rr
    step()
    t, it, rr = step()
    total = sum(t.values())
    report("C3+step", "picard_viscous_step", total, N, None, None,
           "; ".join(f"{k} {v:.1f} ms" for k, v in t.items()) + f"; PCG {it} its (relres {rr:.1e}), FP32 cph V-cycle")


def run_c5(reps):
    m = bfs()
    ctx = Context(m, 3, visc_law=C5_LAW)
    N = ctx.n_dofs() * 3
    ulin = dev(c5_linearization(m, 3))
    ms = timeit(lambda: ctx.update_viscosity(ulin), 5, reps)
    report("C5", "update_viscosity", ms, N, 8 * m.n_cells * (3 * 64 + 64 + 6 * 16))
    src = dev(uniform(0, N))
    dst = torch.empty_like(src)
    ms = timeit(lambda: ctx.apply_viscous(src, dst), 20, reps)
    report("C5", "apply_viscous", ms, N, visc_bytes(m.n_cells, 4, False), visc_flops(N, 4, False))
    # the BFS viscous step's preconditioner: V-cycle 3 -> 2 -> 1 (FP64 and FP32 levels), mass 1e3
    ctx2 = Context(m, 3, visc_law=C5_LAW, degrees=[3, 2, 1])
    ctx2.set_mass(A.OP_VISCOUS, 1.0e3)
    ctx2.update_viscosity(ulin)
    lams = [1.2 * ctx2.estimate_lambda_max(A.OP_VISCOUS, dev(uniform(2, 3 * ctx2.n_dofs(l))), level=l, steps=15)
            for l in range(3)]
    x = torch.zeros_like(src)
    # where the V-cycle's time goes: the Helmholtz apply and Chebyshev(5) from zero on each p-level
    for l, kk in enumerate((3, 2, 1)):
        Nl = 3 * ctx2.n_dofs(l)
        sl, dl = dev(uniform(3 + l, Nl)), torch.empty(Nl, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: ctx2.apply_viscous(sl, dl, level=l), 20, reps)
        report("C5", f"level{l}_k{kk}_apply_helmholtz", ms, Nl, visc_bytes(m.n_cells, kk + 1, False),
               visc_flops(Nl, kk + 1, False))
        wk = torch.empty(2 * Nl, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: ctx2.chebyshev_smooth(A.OP_VISCOUS, dl, sl, lams[l] / 20.0, lams[l], degree=5,
                                                  x_is_zero=True, work=wk, level=l), 5, reps)
        report("C5", f"level{l}_k{kk}_chebyshev5_from_zero", ms, Nl, None, None, "4 applies with fused epilogue + first step")
        del sl, dl, wk
    ms = timeit(lambda: ctx2.vcycle(A.OP_VISCOUS, src, x, lams), 5, reps)
    report("C5", "viscous_vcycle_3_2_1", ms, N, None, None, "Helmholtz (mass 1e3) Carreau V-cycle, FP64 levels")
    ms = timeit(lambda: ctx2.vcycle_fp32(A.OP_VISCOUS, src, x, lams), 5, reps)
    report("C5", "viscous_vcycle_fp32_3_2_1", ms, N, None, None, "FP32 levels")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5,f1,f2")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for c in a.configs.split(","):
        {"2": run_c2, "3": run_c3, "4": run_c4, "5": run_c5, "f1": run_f1, "f2": run_f2, "f4": run_f4, "f3": run_f3, "step": run_step}[c](a.reps)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
