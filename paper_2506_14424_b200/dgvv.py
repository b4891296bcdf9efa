"""Python binding of the dgvv C ABI (include/dgvv.h) — argument marshalling only.

Vectors are torch CUDA float64 tensors (contiguous, canonical layout); every call forwards
raw device pointers and the current torch CUDA stream to libdgvv.so, whose kernels do all
of the work.  Laws are given as dicts and packed into dgvv_law.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi as A


def pack_law(law):
    """dict -> dgvv_law (marshalling: kind + parameter slots as documented in dgvv.h)."""
    if law is None:
        return None
    L = A.DgvvLaw()
    k = law["kind"]
    if k == "const":
        L.kind, vals = A.LAW_CONST, [law["value"]]
    elif k == "sin3":
        L.kind, vals = A.LAW_SIN3, [law.get("mean", 1.0), law.get("amp", 0.5)]
    elif k == "exp":
        L.kind, vals = A.LAW_EXP, [law["rate"]]
    elif k == "carreau":
        L.kind, vals = A.LAW_CARREAU, [law["eta0"], law["eta_inf"], law["lam"], law["n"]]
    else:
        raise ValueError(f"law kind {k!r} has no dgvv_law encoding")
    for i, v in enumerate(vals):
        L.p[i] = float(v)
    return L


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor, n: int | None = None, name="vector"):
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous CUDA float64 tensor")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name}: expected {n} entries, got {t.numel()}")
    return C.c_void_p(t.data_ptr())


class Context:
    """One dgvv context (one mesh partition, a hierarchy of degrees, up to two operators)."""

    def __init__(self, mesh, degree: int, visc_law=None, poisson_law=None, degrees=None, ip=1.0,
                 formulation="divergence", nccl_comm=None, n_ghost=0, ghost_global_id=None,
                 ghost_owner=None, first_global_cell=0, n_owned=None):
        L = A.lib()
        self._L = L
        n_owned = mesh.n_cells if n_owned is None else n_owned
        self.n_ghost = int(n_ghost)
        self._nb = np.ascontiguousarray(mesh.neighbor, dtype=np.int64)
        if self._nb.shape != (n_owned + n_ghost, 6):                  # the C ABI reads this many rows
            raise ValueError(f"mesh.neighbor: expected ({n_owned + n_ghost}, 6), got {self._nb.shape}")
        self._nodes = np.ascontiguousarray(mesh.nodes, dtype=np.float64)
        m = A.DgvvMesh()
        m.n_cells = n_owned
        m.n_ghost = n_ghost
        m.first_global_cell = first_global_cell
        m.neighbor = self._nb.ctypes.data_as(C.POINTER(C.c_int64))
        if n_ghost:
            self._gid = np.ascontiguousarray(ghost_global_id, dtype=np.int64)
            self._gown = np.ascontiguousarray(ghost_owner, dtype=np.int32)
            m.ghost_global_id = self._gid.ctypes.data_as(C.POINTER(C.c_int64))
            m.ghost_owner = self._gown.ctypes.data_as(C.POINTER(C.c_int32))
        m.map_degree = mesh.map_degree
        m.nodes = self._nodes.ctypes.data_as(C.POINTER(C.c_double))
        degs = [degree] if degrees is None else list(degrees)
        self.degrees = degs
        self._degs = (C.c_int32 * len(degs))(*degs)
        o = A.DgvvOptions()
        o.n_levels = len(degs)
        o.degrees = self._degs
        o.ip_factor = ip
        o.formulation = A.FORM_DIVERGENCE if formulation == "divergence" else A.FORM_LAPLACE
        o.nccl_comm = nccl_comm
        self._vl, self._pl = pack_law(visc_law), pack_law(poisson_law)
        h = C.c_void_p()
        A.check(L.dgvv_setup(C.byref(m), degree,
                             C.byref(self._vl) if self._vl is not None else None,
                             C.byref(self._pl) if self._pl is not None else None,
                             C.byref(o), _stream(), C.byref(h)))
        self.h = h
        self.n_owned = n_owned

    def close(self):
        if getattr(self, "h", None):
            self._L.dgvv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ sizes
    def n_dofs(self, level=0):
        nl, ng = C.c_int64(), C.c_int64()
        A.check(self._L.dgvv_sizes(self.h, level, C.byref(nl), C.byref(ng)))
        return nl.value

    def n_global_dofs(self, level=0):
        nl, ng = C.c_int64(), C.c_int64()
        A.check(self._L.dgvv_sizes(self.h, level, C.byref(nl), C.byref(ng)))
        return ng.value

    def _n(self, op, level):
        return (1 if op == A.OP_POISSON else 3) * self.n_dofs(level)

    # ------------------------------------------------------------------ calls
    def update_viscosity(self, u_lin):
        A.check(self._L.dgvv_update_viscosity(self.h, _ptr(u_lin, self._n(0, 0), "u_lin"), _stream()))
        self._ulin = u_lin          # the library borrows u_lin until the next update

    def apply_viscous(self, src, dst, level=0):
        n = self._n(A.OP_VISCOUS, level)
        A.check(self._L.dgvv_apply_viscous(self.h, level, _ptr(src, n, "src"), _ptr(dst, n, "dst"), _stream()))
        return dst

    def apply_viscous_host(self, src_host, dst_host, level=0):
        """dst_host = A_visc src_host with host (CPU, preferably pinned) tensors; the copies are
        pipelined with the apply inside the library (dgvv_apply_viscous_host)."""
        n = self._n(A.OP_VISCOUS, level)
        for t, nm in ((src_host, "src_host"), (dst_host, "dst_host")):
            if t.device.type != "cpu" or t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != n:
                raise ValueError(f"{nm}: contiguous float64 CPU tensor of {n} entries required")
        A.check(self._L.dgvv_apply_viscous_host(self.h, level, C.c_void_p(src_host.data_ptr()),
                                                C.c_void_p(dst_host.data_ptr()), _stream()))
        return dst_host

    def apply_linearized_viscous(self, src, dst):
        n = self._n(A.OP_VISCOUS, 0)
        A.check(self._L.dgvv_apply_linearized_viscous(self.h, _ptr(src, n, "src"), _ptr(dst, n, "dst"), _stream()))
        return dst

    def apply_poisson(self, src, dst, level=0):
        n = self._n(A.OP_POISSON, level)
        A.check(self._L.dgvv_apply_poisson(self.h, level, _ptr(src, n, "src"), _ptr(dst, n, "dst"), _stream()))
        return dst

    def inverse_diagonal(self, op, dst, level=0):
        A.check(self._L.dgvv_inverse_diagonal(self.h, op, level, _ptr(dst, self._n(op, level), "dst"), _stream()))
        return dst

    def estimate_lambda_max(self, op, v0, level=0, steps=20):
        out = C.c_double()
        A.check(self._L.dgvv_estimate_lambda_max(self.h, op, level, steps, _ptr(v0, self._n(op, level), "v0"),
                                                 C.byref(out), _stream()))
        return out.value

    def chebyshev_smooth(self, op, x, b, lam_lo, lam_hi, degree=5, x_is_zero=False, work=None, level=0):
        n = self._n(op, level)
        if work is None:
            work = torch.empty(2 * n, dtype=torch.float64, device=x.device)
        A.check(self._L.dgvv_chebyshev_smooth(self.h, op, level, _ptr(x, n, "x"), _ptr(b, n, "b"), degree,
                                              lam_lo, lam_hi, int(x_is_zero), _ptr(work, 2 * n, "work"), _stream()))
        return x

    def prolongate(self, op, fine_level, coarse, fine, beta=0.0):
        A.check(self._L.dgvv_prolongate(self.h, op, fine_level, _ptr(coarse, self._n(op, fine_level + 1), "coarse"),
                                        _ptr(fine, self._n(op, fine_level), "fine"), beta, _stream()))
        return fine

    def restrict(self, op, fine_level, fine, coarse, beta=0.0):
        A.check(self._L.dgvv_restrict(self.h, op, fine_level, _ptr(fine, self._n(op, fine_level), "fine"),
                                      _ptr(coarse, self._n(op, fine_level + 1), "coarse"), beta, _stream()))
        return coarse

    def vcycle(self, op, b, x, lam_hi_per_level):
        n = self._n(op, 0)
        arr = self._lams(lam_hi_per_level)
        A.check(self._L.dgvv_vcycle(self.h, op, _ptr(b, n, "b"), _ptr(x, n, "x"), arr, _stream()))
        return x

    def set_mass(self, op, mass):
        """Helmholtz form mass * M + A_op for every later call on op (dgvv_set_mass)."""
        A.check(self._L.dgvv_set_mass(self.h, op, float(mass)))

    def cg_solve(self, op, b, x, rtol=1e-8, maxit=200, precond="vcycle", lam_hi_per_level=None):
        """Preconditioned CG on level 0 (dgvv_cg_solve); x = initial guess in, solution out.
        precond: "none", "jacobi", "vcycle" or "vcycle_fp32".  Returns (iterations, ||r|| / ||b||)."""
        n = self._n(op, 0)
        pc = {"none": A.PRECOND_NONE, "jacobi": A.PRECOND_JACOBI, "vcycle": A.PRECOND_VCYCLE,
              "vcycle_fp32": A.PRECOND_VCYCLE_FP32}[precond]
        arr = None
        if lam_hi_per_level is not None:
            arr = self._lams(lam_hi_per_level)
        it, rr = C.c_int32(), C.c_double()
        A.check(self._L.dgvv_cg_solve(self.h, op, _ptr(b, n, "b"), _ptr(x, n, "x"), float(rtol), int(maxit), pc,
                                      arr, C.byref(it), C.byref(rr), _stream()))
        return it.value, rr.value

    def vcycle_fp32(self, op, b, x, lam_hi_per_level):
        """x = V(b) with all multigrid levels in FP32 (dgvv_vcycle_fp32); b, x FP64 device vectors."""
        n = self._n(op, 0)
        arr = self._lams(lam_hi_per_level)
        A.check(self._L.dgvv_vcycle_fp32(self.h, op, _ptr(b, n, "b"), _ptr(x, n, "x"), arr, _stream()))
        return x

    def set_penalty_parameters(self, tau_div, tau_cont):
        """Per-cell penalty parameters (owned cells, then ghosts in mesh ghost order) of the
        penalty-step operator (dgvv_set_penalty_parameters)."""
        td = np.ascontiguousarray(tau_div, dtype=np.float64)
        tc = np.ascontiguousarray(tau_cont, dtype=np.float64)
        nt = self.n_owned + self.n_ghost                             # the C ABI reads n_cells + n_ghost entries
        if td.shape != (nt,) or tc.shape != (nt,):
            raise ValueError(f"tau_div/tau_cont: expected {nt} entries each, got {td.shape} / {tc.shape}")
        A.check(self._L.dgvv_set_penalty_parameters(self.h, td.ctypes.data_as(C.POINTER(C.c_double)),
                                                    tc.ctypes.data_as(C.POINTER(C.c_double))))

    def apply_penalty(self, src, dst, level=0):
        n = 3 * self.n_dofs(level)
        if level == 0:
            A.check(self._L.dgvv_apply_penalty(self.h, _ptr(src, n, "src"), _ptr(dst, n, "dst"), _stream()))
        else:
            A.check(self._L.dgvv_apply_penalty_level(self.h, level, _ptr(src, n, "src"), _ptr(dst, n, "dst"),
                                                     _stream()))
        return dst

    def set_transport(self, w):
        """Transport field w of the convective term (dgvv_set_transport; level-0 vector, copied)."""
        A.check(self._L.dgvv_set_transport(self.h, _ptr(w, 3 * self.n_dofs(0), "w"), _stream()))

    def apply_convective(self, src, dst):
        """dst = C(w) src, the upwind DG convective term (dgvv_apply_convective)."""
        n = 3 * self.n_dofs(0)
        A.check(self._L.dgvv_apply_convective(self.h, _ptr(src, n, "src"), _ptr(dst, n, "dst"), _stream()))
        return dst

    def apply_oseen(self, src, dst, alpha_c=1.0):
        """dst = (mass M + A(nu) + alpha_c C(w)) src (dgvv_apply_oseen)."""
        n = 3 * self.n_dofs(0)
        A.check(self._L.dgvv_apply_oseen(self.h, float(alpha_c), _ptr(src, n, "src"), _ptr(dst, n, "dst"),
                                         _stream()))
        return dst

    def gmres_solve(self, b, x, alpha_c=1.0, rtol=1e-8, restart=30, maxit=300, precond="vcycle",
                    lam_hi_per_level=None):
        """Right-preconditioned restarted GMRES on mass M + A(nu) + alpha_c C(w) (dgvv_gmres_solve);
        x = initial guess in, solution out.  Returns (iterations, ||b - A x|| / ||b||)."""
        n = 3 * self.n_dofs(0)
        pc = {"none": A.PRECOND_NONE, "jacobi": A.PRECOND_JACOBI, "vcycle": A.PRECOND_VCYCLE,
              "vcycle_fp32": A.PRECOND_VCYCLE_FP32}[precond]
        arr = None
        if lam_hi_per_level is not None:
            arr = self._lams(lam_hi_per_level)
        it, rr = C.c_int32(), C.c_double()
        A.check(self._L.dgvv_gmres_solve(self.h, float(alpha_c), _ptr(b, n, "b"), _ptr(x, n, "x"), float(rtol),
                                         int(restart), int(maxit), pc, arr, C.byref(it), C.byref(rr), _stream()))
        return it.value, rr.value

    def chain_levels(self):
        """Number of multigrid levels of the chain: own p-levels, then either the continuous levels
        of this and every coarse context (c-level enabled) or the coarse contexts' chains."""
        if getattr(self, "_continuous", False):
            c, n = self, len(self.degrees)
            while c is not None:
                n += 1
                c = getattr(c, "_coarse", None)
            return n
        c, n = self, 0
        while c is not None:
            if getattr(c, "_continuous", False):
                return n + c.chain_levels()
            n += len(c.degrees)
            c = getattr(c, "_coarse", None)
        return n

    def set_continuous_level(self, enable=True):
        """Enable the continuous Q1 (c-) level below the coarsest (degree-1) DG level
        (dgvv_set_continuous_level).  Returns (vertices, colours)."""
        A.check(self._L.dgvv_set_continuous_level(self.h, int(bool(enable))))
        self._continuous = bool(enable)
        if not enable:
            return None
        nv, ncol = C.c_int32(), C.c_int32()
        A.check(self._L.dgvv_continuous_level_info(self.h, C.byref(nv), C.byref(ncol)))
        self.n_vertices = nv.value
        return nv.value, ncol.value

    def apply_continuous(self, op, src, dst):
        n = (3 if op == A.OP_VISCOUS else 1) * self.n_vertices
        A.check(self._L.dgvv_apply_continuous(self.h, op, _ptr(src, n, "src"), _ptr(dst, n, "dst"), _stream()))
        return dst

    def embed_continuous(self, op, src, dst, transpose=False, beta=0.0):
        nc = 3 if op == A.OP_VISCOUS else 1
        n_cg, n_dg = nc * self.n_vertices, nc * 8 * self.n_owned      # Q1 vertices / DG_1 cells
        n_src, n_dst = (n_dg, n_cg) if transpose else (n_cg, n_dg)
        A.check(self._L.dgvv_embed_continuous(self.h, op, int(bool(transpose)), _ptr(src, n_src, "src"),
                                              _ptr(dst, n_dst, "dst"), float(beta), _stream()))
        return dst

    def estimate_lambda_max_continuous(self, op, v0, steps=20):
        """lambda_max(D^-1 A) of the continuous level (dgvv_estimate_lambda_max, level = n_levels)."""
        out = C.c_double()
        n = (3 if op == A.OP_VISCOUS else 1) * self.n_vertices
        A.check(self._L.dgvv_estimate_lambda_max(self.h, op, len(self.degrees), steps, _ptr(v0, n, "v0"),
                                                 C.byref(out), _stream()))
        return out.value

    def _lams(self, lam_hi_per_level):
        lam = [float(v) for v in lam_hi_per_level]
        if len(lam) < self.chain_levels():
            raise ValueError(f"lam_hi_per_level: {len(lam)} values for {self.chain_levels()} levels")
        return (C.c_double * len(lam))(*lam)

    def set_coarse_context(self, coarse, parent, octant):
        """Append the levels of `coarse` below this context's coarsest level (h-coarsening,
        dgvv_set_coarse_context); parent/octant per fine cell.  Keeps a reference to `coarse`."""
        par = np.ascontiguousarray(parent, dtype=np.int32)
        octa = np.ascontiguousarray(octant, dtype=np.int8)
        if par.shape != (self.n_owned,) or octa.shape != (self.n_owned,):   # the C ABI reads n_cells entries
            raise ValueError(f"parent/octant: expected {self.n_owned} entries each, got {par.shape} / {octa.shape}")
        A.check(self._L.dgvv_set_coarse_context(self.h, coarse.h, par.ctypes.data_as(C.POINTER(C.c_int32)),
                                                octa.ctypes.data_as(C.POINTER(C.c_int8))))
        self._coarse = coarse

    def prolongate_h(self, op, coarse_vec, fine_vec, beta=0.0):
        nf = self._n(op, len(self.degrees) - 1)
        nc = self._coarse._n(op, 0) if getattr(self, "_coarse", None) is not None else None
        A.check(self._L.dgvv_prolongate_h(self.h, op, _ptr(coarse_vec, nc, "coarse"), _ptr(fine_vec, nf, "fine"),
                                          float(beta), _stream()))
        return fine_vec

    def restrict_h(self, op, fine_vec, coarse_vec, beta=0.0):
        nf = self._n(op, len(self.degrees) - 1)
        nc = self._coarse._n(op, 0) if getattr(self, "_coarse", None) is not None else None
        A.check(self._L.dgvv_restrict_h(self.h, op, _ptr(fine_vec, nf, "fine"), _ptr(coarse_vec, nc, "coarse"),
                                        float(beta), _stream()))
        return coarse_vec

    def setup_coarse_solver(self, op):
        """Dense direct solve on the coarsest level (dgvv_setup_coarse_solver); returns its size."""
        n = C.c_int32()
        A.check(self._L.dgvv_setup_coarse_solver(self.h, op, C.byref(n)))
        return n.value

    def dot(self, a, b, ncomp=1, level=0):
        out = C.c_double()
        n = ncomp * self.n_dofs(level)
        A.check(self._L.dgvv_dot(self.h, level, ncomp, _ptr(a, n, "a"), _ptr(b, n, "b"), C.byref(out), _stream()))
        return out.value

    # ------------------------------------------------------------------ ghosts (multi-GPU)
    def exchange_bytes(self, op=0, level=0):
        """(sent, received) bytes of one apply's face-trace exchange (dgvv_exchange_bytes)."""
        a, b = C.c_int64(), C.c_int64()
        A.check(self._L.dgvv_exchange_bytes(self.h, level, op, C.byref(a), C.byref(b)))
        return a.value, b.value

    def ghost_layout(self):
        """[(peer rank, send count, recv count)] in peer order."""
        n = C.c_int32()
        A.check(self._L.dgvv_ghost_layout(self.h, C.byref(n), None, None, None))
        r, sc, rc = (C.c_int32 * max(1, n.value))(), (C.c_int32 * max(1, n.value))(), (C.c_int32 * max(1, n.value))()
        A.check(self._L.dgvv_ghost_layout(self.h, C.byref(n), r, sc, rc))
        return [(r[i], sc[i], rc[i]) for i in range(n.value)]

    def pack_ghosts(self, kind, src, sendbuf, level=0):
        k = self.degrees[level]
        per = (1 if kind == A.GHOST_POISSON else 3) * (k + 1) ** 3
        n_send = sum(s for _, s, _ in self.ghost_layout())
        A.check(self._L.dgvv_pack_ghosts(self.h, level, kind, _ptr(src, per * self.n_owned, "src"),
                                         _ptr(sendbuf, max(1, per * n_send) if n_send else None, "sendbuf"),
                                         _stream()))
        return sendbuf

    def ghost_buffer(self, kind, n_ghost, level=0):
        """torch view (no copy) of the library-owned ghost buffer of `kind`."""
        p = C.c_void_p()
        A.check(self._L.dgvv_ghost_buffer(self.h, level, kind, C.byref(p)))
        k = self.degrees[level]
        per = (1 if kind == A.GHOST_POISSON else 3) * (k + 1) ** 3   # TRANSPORT: 3 components
        return _wrap_device(p.value, n_ghost * per)

    def coefficient_range(self, op, level=0):
        lo, hi = C.c_double(), C.c_double()
        A.check(self._L.dgvv_coefficient_range(self.h, op, level, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value


def _wrap_device(ptr: int, n: int) -> torch.Tensor:
    """Non-owning float64 CUDA tensor over library memory (marshalling for the ghost buffers)."""
    class _Iface:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_Iface(), device="cuda")


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    A.check(A.lib().dgvv_nccl_get_unique_id(buf))
    return buf.raw


def nccl_comm_init(uid: bytes, nranks: int, rank: int):
    comm = C.c_void_p()
    A.check(A.lib().dgvv_nccl_comm_init(uid, nranks, rank, C.byref(comm)))
    return comm


class ThreadGroup:
    """In-process communicator group of R ranks (dgvv_thread_group_create): rank r's communicator
    (comm(r)) is passed to Context(nccl_comm=...) like an NCCL one; each rank is driven by its own
    host thread on its own CUDA stream (see include/dgvv.h)."""

    def __init__(self, nranks: int):
        g = C.c_void_p()
        A.check(A.lib().dgvv_thread_group_create(int(nranks), C.byref(g)))
        self.h, self.nranks = g, int(nranks)

    def comm(self, rank: int):
        cm = C.c_void_p()
        A.check(A.lib().dgvv_thread_group_comm(self.h, int(rank), C.byref(cm)))
        return cm

    def close(self):
        if self.h:
            A.lib().dgvv_thread_group_destroy(self.h)
            self.h = None
