"""DG discretisation, geometry and the SIPG operator applications (oracle).
Test infrastructure only — see oracle/__init__.py.

What is computed (full-tensor quadrature, no sum factorisation):
  * viscous_apply  — the SIPG viscous form v_h^e summed over all cells
    (§4.1, eqn:viscous_term_weak) with the fluxes of PAPER.md:1088-1111
    (u^dag = {{u}}, tau1^dag = {{nu grad u}} - tau [[u]], tau2^dag = (tau1^dag)^T), mirror
    boundary conditions (reading G7), written per face as SURVEY.md
    Appendix A.1.  Output y[K,c,i] = a(e_c phi_i^K, u; nu).
  * poisson_apply  — the SIPG Poisson form of PAPER.md:713-758 (eqn:pressure_step_weak) with
    a coefficient c multiplying grad p (reading G16) and the penalty sign of reading G4,
    written per face as SURVEY.md Appendix A.2.
Conventions: G1 Gauss n_q = k+1; G2 Lagrange basis on the Gauss points;
G3 tau = IP (k+1)^2 max(H-,H+) nu_F, H_K = (A(dK\\Gamma)/2 + A(dK cap Gamma)) / V(K);
G5 symmetrised penalty; G6 nu_F = (nu- + nu+)/2, each side's own nu in its consistency
term; G8 nu pointwise at quadrature points, face values from each side; G11 K- = lower
global id, n and dA from K-.  Reference cell [0,1]^3.  Canonical vector layout
[cell][component][z][y][x].
"""
from __future__ import annotations

import numpy as np

from . import basis as B
from . import laws


class Disc:
    """Tabulations + geometry for one mesh and DG degree k (velocity or pressure space)."""

    def __init__(self, mesh, k: int, ip: float = 1.0):
        self.mesh = mesh
        self.k = k
        self.n = n = k + 1
        self.N = n ** 3
        self.P = n * n
        self.ip = ip
        self.xi, self.w1 = B.gauss01(n)
        self.vol_pts = B.tensor_points(self.xi)
        self.vol_w = B.tensor_weights(self.w1)
        self.Phi, self.dPhi = B.tabulate(self.xi, self.vol_pts)
        self.face_pts = [B.face_points(self.xi, f) for f in range(6)]
        self.face_w = B.face_weights(self.w1)
        tf = [B.tabulate(self.xi, p) for p in self.face_pts]
        self.PhiF = [t[0] for t in tf]
        self.dPhiF = [t[1] for t in tf]
        gn = B.gll01(mesh.map_degree)
        self.G, self.dG = B.tabulate(gn, self.vol_pts)
        tg = [B.tabulate(gn, p) for p in self.face_pts]
        self.GF = [t[0] for t in tg]
        self.dGF = [t[1] for t in tg]
        cen = [B.face_points(np.array([0.5]), f) for f in range(6)]
        self.Gcen = [B.tabulate(gn, c)[0] for c in cen]
        self.periods = np.asarray(mesh.periods, dtype=np.float64)

    # ------------------------------------------------------------------ geometry
    def _map(self, cells, G, dG):
        X = self.mesh.nodes[cells]                                  # [C, M, 3]
        x = np.einsum("pm,cmi->cpi", G, X)
        J = np.einsum("dpm,cmi->cpid", dG, X)                       # J[c,p,i,d] = dx_i/dxi_d
        detJ = np.linalg.det(J)
        if np.any(detJ <= 0):
            raise ValueError("non-positive Jacobian")
        Jinv = np.linalg.inv(J)                                     # Jinv[c,p,d,i] = dxi_d/dx_i
        return x, detJ, Jinv

    def vol_geom(self, cells):
        """x [C,Q,3], JxW [C,Q], Jinv [C,Q,3,3] at the cell quadrature points."""
        x, detJ, Jinv = self._map(cells, self.G, self.dG)
        return x, detJ * self.vol_w, Jinv

    def face_geom(self, cells, f):
        """x, Jinv, outward unit normal n and dA at the points of local face f (Nanson:
        n dA = det J J^-T N dA_ref)."""
        x, detJ, Jinv = self._map(cells, self.GF[f], self.dGF[f])
        d, s = f // 2, f % 2
        v = (2.0 * s - 1.0) * Jinv[:, :, d, :]                      # J^-T N
        ln = np.linalg.norm(v, axis=-1)
        return x, Jinv, v / ln[..., None], detJ * ln * self.face_w

    def face_centroid(self, cells, f):
        return np.einsum("pm,cmi->cpi", self.Gcen[f], self.mesh.nodes[cells])[:, 0, :]

    def H(self, cells):
        """Penalty length scale H_K = (A(dK\\Gamma)/2 + A(dK cap Gamma)) / V(K) (G3)."""
        cells = np.asarray(cells)
        _, JxW, _ = self.vol_geom(cells)
        V = JxW.sum(axis=1)
        num = np.zeros(len(cells))
        for f in range(6):
            A = self.face_geom(cells, f)[3].sum(axis=1)
            bnd = self.mesh.neighbor[cells, f] < 0
            num += np.where(bnd, A, 0.5 * A)
        return num / V

    # ------------------------------------------------------------ face pairing
    def _periodic_shift_ok(self, dx, scale):
        """dx [F,3] = centroid difference; accepted if each component is 0 or +-period."""
        tol = 1e-8 * scale
        ok = np.ones(len(dx), dtype=bool)
        for d in range(3):
            L = self.periods[d]
            c = np.abs(dx[:, d]) < tol
            if L > 0:
                c |= np.abs(np.abs(dx[:, d]) - L) < tol
            ok &= c
        return ok

    def match_faces(self, a, fa, b):
        """For faces (a[i], fa) with neighbour cells b[i]: find b's face fb touching a[i]
        (geometrically, centroids equal modulo periods) and the permutation perm[i, p] of b's
        face points matching a's face point p.  Returns fb [F], perm [F, P], shift [F, 3]."""
        a, b = np.asarray(a), np.asarray(b)
        F = len(a)
        xa_c = self.face_centroid(a, fa)
        scale = np.linalg.norm(self.mesh.nodes[a, -1] - self.mesh.nodes[a, 0], axis=-1)
        fb = np.full(F, -1)
        shift = np.zeros((F, 3))
        for g in range(6):
            cand = (self.mesh.neighbor[b, g] == a) & (fb < 0)
            if not np.any(cand):
                continue
            xb_c = self.face_centroid(b[cand], g)
            dx = xa_c[cand] - xb_c
            ok = self._periodic_shift_ok(dx, scale[cand])
            idx = np.nonzero(cand)[0][ok]
            fb[idx] = g
            shift[idx] = dx[ok]
        if np.any(fb < 0):
            raise ValueError("face pairing failed: neighbour table and geometry disagree")
        perm = np.empty((F, self.P), dtype=np.int64)
        xa = self.face_geom(a, fa)[0]
        for g in range(6):
            sel = fb == g
            if not np.any(sel):
                continue
            xb = self.face_geom(b[sel], g)[0] + shift[sel][:, None, :]
            dist = np.linalg.norm(xa[sel][:, :, None, :] - xb[:, None, :, :], axis=-1)
            p = np.argmin(dist, axis=2)
            dmin = np.take_along_axis(dist, p[:, :, None], axis=2)[..., 0]
            if np.any(dmin > 1e-9 * scale[sel][:, None]):
                raise ValueError("face quadrature points do not coincide")
            perm[sel] = p
        return fb, perm, shift

    def unique_faces(self, cells):
        """All faces touching `cells`: interior faces once as (K-, f-, K+) with K- < K+
        (G11), and boundary faces (K, f, bc)."""
        nb = self.mesh.neighbor
        cells = np.asarray(cells)
        inter = {}
        bnd = []
        for f in range(6):
            o = nb[cells, f]
            for c, t in zip(cells[o < 0], o[o < 0]):
                bnd.append((int(c), f, int(-1 - t)))
            sel = o >= 0
            cs, ts = cells[sel], o[sel]
            lo = cs < ts
            for c, t in zip(cs[lo], ts[lo]):
                inter[(int(c), f)] = int(t)
            hi = ~lo
            if np.any(hi):
                # face seen from K+: identify K-'s local face geometrically
                fb, _, _ = self.match_faces(cs[hi], f, ts[hi])
                for c, t, g in zip(cs[hi], ts[hi], fb):
                    inter[(int(t), int(g))] = int(c)
        return inter, bnd


# ---------------------------------------------------------------------- viscosity at points
class AnalyticNu:
    """Coefficient evaluated pointwise at the mapped quadrature points (G8)."""

    def __init__(self, disc: Disc, law: dict):
        self.d, self.law = disc, law

    def vol(self, cells):
        return laws.analytic(self.law, self.d.vol_geom(cells)[0])

    def face(self, cells, f):
        return laws.analytic(self.law, self.d.face_geom(cells, f)[0])


class ArrayNu:
    """Explicit point values: vol [n_cells, Q], face [n_cells, 6, P] (own-side values at own points)."""

    def __init__(self, vol, face):
        self.v, self.f = vol, face

    def vol(self, cells):
        return self.v[cells]

    def face(self, cells, f):
        return self.f[cells, f]


def grad_at(disc, U, dPhi, Jinv):
    """Physical gradient of a vector field with coefficients U [C,3,N] at points with
    reference-derivative tabulation dPhi [3,P,N]: G[c,p,i,j] = d u_i / d x_j."""
    gxi = np.einsum("dpn,cin->cpid", dPhi, U)
    return np.einsum("cpid,cpdj->cpij", gxi, Jinv)


def sym(G):
    return 0.5 * (G + np.swapaxes(G, -1, -2))


class CarreauNu:
    """nu = eta(gamma_dot(eps(u_lin))) at every cell point and, per side, at every face point
    from that side's own trace gradient (PAPER.md:838-866 eqn:viscosity_pointwise; G8, G9)."""

    def __init__(self, disc: Disc, u_lin: np.ndarray, p: dict):
        self.d, self.p = disc, p
        self.U = u_lin.reshape(disc.mesh.n_cells, 3, disc.N)

    def _eta(self, eps):
        p = self.p
        return laws.carreau(laws.shear_rate(eps), p["eta0"], p["eta_inf"], p["lam"], p["n"])

    def vol(self, cells):
        _, _, Jinv = self.d.vol_geom(cells)
        return self._eta(sym(grad_at(self.d, self.U[cells], self.d.dPhi, Jinv)))

    def face(self, cells, f):
        _, Jinv, _, _ = self.d.face_geom(cells, f)
        return self._eta(sym(grad_at(self.d, self.U[cells], self.d.dPhiF[f], Jinv)))


def coarse_level_ulin(disc_f: Disc, disc_c: Disc, u_lin: np.ndarray) -> np.ndarray:
    """Reading G19 (§5.3: the viscosity is stored at the integration points
    of every multigrid level and refreshed on all levels when the linearisation changes): the
    linearisation velocity of a coarser p-level is the fine polynomial u_lin evaluated at that
    level's Gauss points, i.e. its coefficients in the coarse collocation basis (G2).  Full-tensor:
    every fine basis function tabulated at every coarse volume point."""
    Phi_fc = B.tabulate(disc_f.xi, disc_c.vol_pts)[0]                  # [N_c, N_f]
    U = u_lin.reshape(disc_f.mesh.n_cells, 3, disc_f.N)
    return np.einsum("pn,cin->cip", Phi_fc, U).reshape(-1)


def coarse_level_nu(disc_f: Disc, disc_c: Disc, u_lin: np.ndarray, p: dict) -> "CarreauNu":
    """G19: the Carreau viscosity of a coarser level, eta(gamma_dot(eps)) of the interpolated
    linearisation velocity at that level's cell points and, per side, its face points (G8)."""
    return CarreauNu(disc_c, coarse_level_ulin(disc_f, disc_c, u_lin), p)


class NewtonDeltaNu:
    """delta nu[w] = 2 g(gamma_dot_0) eps(u0):eps(w), g = eta'/gamma_dot (reading G10), at every
    cell point and per side at face points from each side's own traces."""

    def __init__(self, disc: Disc, u0: np.ndarray, w: np.ndarray, p: dict):
        self.d, self.p = disc, p
        self.U0 = u0.reshape(disc.mesh.n_cells, 3, disc.N)
        self.W = w.reshape(disc.mesh.n_cells, 3, disc.N)

    def _dnu(self, e0, ew):
        p = self.p
        g = laws.carreau_g(laws.shear_rate(e0), p["eta0"], p["eta_inf"], p["lam"], p["n"])
        return 2.0 * g * np.einsum("...ij,...ij->...", e0, ew)

    def vol(self, cells):
        _, _, Jinv = self.d.vol_geom(cells)
        e0 = sym(grad_at(self.d, self.U0[cells], self.d.dPhi, Jinv))
        ew = sym(grad_at(self.d, self.W[cells], self.d.dPhi, Jinv))
        return self._dnu(e0, ew)

    def face(self, cells, f):
        _, Jinv, _, _ = self.d.face_geom(cells, f)
        e0 = sym(grad_at(self.d, self.U0[cells], self.d.dPhiF[f], Jinv))
        ew = sym(grad_at(self.d, self.W[cells], self.d.dPhiF[f], Jinv))
        return self._dnu(e0, ew)


# ---------------------------------------------------------------------- helpers
def _prepare(disc, cells):
    nc = disc.mesh.n_cells
    if cells is None:
        cells = np.arange(nc)
    cells = np.unique(np.asarray(cells, dtype=np.int64))
    row = np.full(nc, -1, dtype=np.int64)
    row[cells] = np.arange(len(cells))
    return cells, row


def _chunks(n, size):
    for s in range(0, n, size):
        yield slice(s, min(n, s + size))


def _group_faces(disc, inter):
    """Group interior faces (K-, f-) -> K+ by (f-, f+); returns dict (fa, fb) -> (a, b, perm)."""
    if not inter:
        return {}
    keys = np.array(list(inter.keys()), dtype=np.int64)
    a_all, fa_all = keys[:, 0], keys[:, 1]
    b_all = np.array(list(inter.values()), dtype=np.int64)
    out = {}
    for fa in range(6):
        s = fa_all == fa
        if not np.any(s):
            continue
        a, b = a_all[s], b_all[s]
        fb, perm, _ = disc.match_faces(a, fa, b)
        for g in range(6):
            t = fb == g
            if np.any(t):
                out[(fa, g)] = (a[t], b[t], perm[t])
    return out


# ---------------------------------------------------------------------- viscous operator
def viscous_apply(disc: Disc, u: np.ndarray, nu, cells=None, formulation: str = "divergence",
                  chunk: int = 4096) -> np.ndarray:
    """y = A(nu) u for the SIPG viscous operator (Appendix A.1 / A.3), rows of `cells` only.

    formulation "divergence": the paper's operator (grad^S in volume and fluxes, penalty
    tau([v].[u] + ([v].n)([u].n)), reading G5).  "laplace": only the tau_1 terms
    (PAPER.md:924-968): volume nu grad v : grad u, fluxes with (1/2) grad, penalty tau [v].[u].
    Returns y [len(cells), 3, N] (cells sorted) or the full vector if cells is None.
    """
    full = cells is None
    d = disc
    nc, N = d.mesh.n_cells, d.N
    U = u.reshape(nc, 3, N)
    cells, row = _prepare(d, cells)
    y = np.zeros((len(cells), 3, N))
    div = formulation == "divergence"
    if formulation not in ("divergence", "laplace"):
        raise ValueError(formulation)
    pen = d.ip * (d.k + 1) ** 2

    # ---- volume: sum_q JxW * [2 nu eps(u) (div) | nu grad u (lap)] : grad v
    for sl in _chunks(len(cells), chunk):
        cs = cells[sl]
        _, JxW, Jinv = d.vol_geom(cs)
        G = grad_at(d, U[cs], d.dPhi, Jinv)                       # [C,Q,3,3]
        nuq = nu.vol(cs)
        S = 2.0 * sym(G) if div else G
        T = (nuq * JxW)[:, :, None, None] * S                      # coefficient of d v_i/d x_j
        # grad v_i = sum_d dPhi[d,q,n] Jinv[q,d,j]
        y[sl] += np.einsum("cqij,dqn,cqdj->cin", T, d.dPhi, Jinv)

    inter, bnd = d.unique_faces(cells)
    # H for every cell touched
    touched = set(cells.tolist())
    for (a, fa), b in inter.items():
        touched.add(a)
        touched.add(b)
    tl = np.array(sorted(touched), dtype=np.int64)
    Hmap = np.zeros(nc)
    Hmap[tl] = d.H(tl)

    def side_eval(cs, f, perm=None):
        x, Jinv, n, dA = d.face_geom(cs, f)
        Uc = U[cs]
        val = np.einsum("pn,cin->cpi", d.PhiF[f], Uc)
        G = grad_at(d, Uc, d.dPhiF[f], Jinv)
        nuf = nu.face(cs, f)
        if perm is not None:
            take = lambda A: np.take_along_axis(A, perm.reshape(perm.shape + (1,) * (A.ndim - 2)), axis=1)
            val, G, nuf, Jinv = take(val), take(G), take(nuf), take(Jinv)
        return val, G, nuf, Jinv, n, dA

    def flux_terms(uj, Gm, Gp, num, nup, n, tau):
        """Value coefficient fv for side '-' and the tensor jn = [u] (x) n (symmetrised for div)."""
        Sm = sym(Gm) if div else 0.5 * Gm
        Sp = sym(Gp) if div else 0.5 * Gp
        sbar = num[..., None, None] * Sm + nup[..., None, None] * Sp
        sbn = np.einsum("cpij,cpj->cpi", sbar, n)
        if div:
            un = np.einsum("cpi,cpi->cp", uj, n)
            pen_v = tau[..., None] * (uj + n * un[..., None])
            jn = sym(uj[..., :, None] * n[..., None, :])
        else:
            pen_v = tau[..., None] * uj
            jn = 0.5 * uj[..., :, None] * n[..., None, :]
        return -sbn + pen_v, jn

    def scatter(cs, f, fv, Gc, Jinv, dA, perm=None):
        """y[cs] += sum_p dA (phi_i fv_c + sum_j Gc_cj d phi_i/d x_j) at the points of face f."""
        Phi, dPhi = d.PhiF[f], d.dPhiF[f]
        if perm is None:
            contrib = np.einsum("cp,pn,cpi->cin", dA, Phi, fv)
            contrib += np.einsum("cp,cpij,dpn,cpdj->cin", dA, Gc, dPhi, Jinv)
        else:
            Phi_p = Phi[perm]                                       # [C,P,N]
            dPhi_p = np.moveaxis(dPhi[:, perm], 0, 1)              # [C,3,P,N]
            contrib = np.einsum("cp,cpn,cpi->cin", dA, Phi_p, fv)
            contrib += np.einsum("cp,cpij,cdpn,cpdj->cin", dA, Gc, dPhi_p, Jinv)
        r = row[cs]
        m = r >= 0
        np.add.at(y, r[m], contrib[m])

    # ---- interior and periodic faces (each once, both sides' test functions)
    for (fa, fb), (a_all, b_all, perm_all) in _group_faces(d, inter).items():
        for sl in _chunks(len(a_all), chunk):
            a, b, perm = a_all[sl], b_all[sl], perm_all[sl]
            ua, Ga, nua, Jia, n, dA = side_eval(a, fa)
            ub, Gb, nub, Jib, _, _ = side_eval(b, fb, perm)
            tau = pen * np.maximum(Hmap[a], Hmap[b])[:, None] * 0.5 * (nua + nub)
            uj = ua - ub
            fv, jn = flux_terms(uj, Ga, Gb, nua, nub, n, tau)
            scatter(a, fa, fv, -nua[..., None, None] * jn, Jia, dA)
            scatter(b, fb, -fv, -nub[..., None, None] * jn, Jib, dA, perm)

    # ---- boundary faces: Dirichlet by the mirror principle (G7), Neumann: no contribution
    bnd = [t for t in bnd if t[2] == 1]
    for f in range(6):
        cs = np.array([c for (c, g, _) in bnd if g == f], dtype=np.int64)
        for sl in _chunks(len(cs), chunk):
            a = cs[sl]
            if len(a) == 0:
                continue
            ua, Ga, nua, Jia, n, dA = side_eval(a, f)
            tau = pen * Hmap[a][:, None] * nua
            uj = 2.0 * ua                                            # u+ = -u-
            fv, jn = flux_terms(uj, Ga, Ga, nua, nua, n, tau)        # grad u+ = grad u-, nu+ = nu-
            scatter(a, f, fv, -nua[..., None, None] * jn, Jia, dA)

    return y.reshape(-1) if full else y


# ---------------------------------------------------------------------- Poisson operator
def poisson_apply(disc: Disc, p: np.ndarray, coef, cells=None, chunk: int = 4096) -> np.ndarray:
    """y = A_P(c) p for the scalar SIPG Poisson form (Appendix A.2):
      volume      sum_q JxW c grad q . grad p
      interior    -[q] (1/2)(c- grad p- + c+ grad p+).n - [p] (1/2)(c- grad q- + c+ grad q+).n + tau [q][p]
      Dirichlet   -q c grad p.n - p c grad q.n + 2 tau q p      (mirror, G7)
    tau = IP (k+1)^2 max(H-,H+) (c- + c+)/2 (G3, G4 sign, G16 coefficient)."""
    full = cells is None
    d = disc
    nc, N = d.mesh.n_cells, d.N
    Pv = p.reshape(nc, N)
    cells, row = _prepare(d, cells)
    y = np.zeros((len(cells), N))
    pen = d.ip * (d.k + 1) ** 2

    for sl in _chunks(len(cells), chunk):
        cs = cells[sl]
        _, JxW, Jinv = d.vol_geom(cs)
        g = np.einsum("dqn,cn,cqdj->cqj", d.dPhi, Pv[cs], Jinv)      # grad p
        cq = coef.vol(cs)
        y[sl] += np.einsum("cq,cqj,dqn,cqdj->cn", cq * JxW, g, d.dPhi, Jinv)

    inter, bnd = d.unique_faces(cells)
    touched = set(cells.tolist())
    for (a, fa), b in inter.items():
        touched.update((a, b))
    tl = np.array(sorted(touched), dtype=np.int64)
    Hmap = np.zeros(nc)
    Hmap[tl] = d.H(tl)

    def side(cs, f, perm=None):
        _, Jinv, n, dA = d.face_geom(cs, f)
        val = np.einsum("pn,cn->cp", d.PhiF[f], Pv[cs])
        g = np.einsum("dpn,cn,cpdj->cpj", d.dPhiF[f], Pv[cs], Jinv)
        cf = coef.face(cs, f)
        Phi, dPhi = d.PhiF[f], d.dPhiF[f]
        if perm is not None:
            val = np.take_along_axis(val, perm, axis=1)
            g = np.take_along_axis(g, perm[..., None], axis=1)
            cf = np.take_along_axis(cf, perm, axis=1)
            Jinv = np.take_along_axis(Jinv, perm[..., None, None], axis=1)
            Phi_c = Phi[perm]
            dPhi_c = np.moveaxis(dPhi[:, perm], 0, 1)
        else:
            Phi_c = np.broadcast_to(Phi, (len(cs),) + Phi.shape)
            dPhi_c = np.broadcast_to(dPhi, (len(cs),) + dPhi.shape)
        # grad phi_i at the points: [C,P,N,3]
        gphi = np.einsum("cdpn,cpdj->cpnj", dPhi_c, Jinv)
        return val, g, cf, Phi_c, gphi, n, dA

    def add(cs, contrib):
        r = row[cs]
        m = r >= 0
        np.add.at(y, r[m], contrib[m])

    for (fa, fb), (a_all, b_all, perm_all) in _group_faces(d, inter).items():
        for sl in _chunks(len(a_all), chunk):
            a, b, perm = a_all[sl], b_all[sl], perm_all[sl]
            pa, ga, ca, Phia, gphia, n, dA = side(a, fa)
            pb, gb, cb, Phib, gphib, _, _ = side(b, fb, perm)
            tau = pen * np.maximum(Hmap[a], Hmap[b])[:, None] * 0.5 * (ca + cb)
            jump = pa - pb
            avg_flux = 0.5 * np.einsum("cpj,cpj->cp", ca[..., None] * ga + cb[..., None] * gb, n)
            # test q- : [q] = q-, grad q- term weighted by c-/2
            add(a, np.einsum("cp,cpn->cn", dA * (-avg_flux + tau * jump), Phia)
                + np.einsum("cp,cpnj,cpj->cn", dA * (-0.5 * ca * jump), gphia, n))
            # test q+ : [q] = -q+, grad q+ term weighted by c+/2
            add(b, np.einsum("cp,cpn->cn", dA * (avg_flux - tau * jump), Phib)
                + np.einsum("cp,cpnj,cpj->cn", dA * (-0.5 * cb * jump), gphib, n))

    for f in range(6):
        cs = np.array([c for (c, g, t) in bnd if g == f and t == 1], dtype=np.int64)
        for sl in _chunks(len(cs), chunk):
            a = cs[sl]
            if len(a) == 0:
                continue
            pa, ga, ca, Phia, gphia, n, dA = side(a, f)
            tau = pen * Hmap[a][:, None] * ca
            dn = np.einsum("cpj,cpj->cp", ga, n)
            add(a, np.einsum("cp,cpn->cn", dA * (-ca * dn + 2.0 * tau * pa), Phia)
                + np.einsum("cp,cpnj,cpj->cn", dA * (-ca * pa), gphia, n))

    return y.reshape(-1) if full else y


# ---------------------------------------------------------------------- Newton linearisation
def newton_apply(disc: Disc, u0: np.ndarray, w: np.ndarray, law: dict, cells=None) -> np.ndarray:
    """J(u0) w = a(., w; nu0) + a(., u0; delta_nu[w])  (reading G10):
    the exact Gateaux derivative of R(u) = a(., u; nu(u)) with nu re-evaluated pointwise at
    every cell and face point (PAPER.md:838-866 for the pointwise law; the paper itself
    Picard-linearises nu)."""
    nu0 = CarreauNu(disc, u0, law)
    dnu = NewtonDeltaNu(disc, u0, w, law)
    return viscous_apply(disc, w, nu0, cells) + viscous_apply(disc, u0, dnu, cells)


def carreau_residual(disc: Disc, u: np.ndarray, law: dict, cells=None) -> np.ndarray:
    """R(u) = a(., u; eta(gamma_dot(u))) — the fully nonlinear viscous term."""
    return viscous_apply(disc, u, CarreauNu(disc, u, law), cells)


def mass_apply(disc: Disc, u: np.ndarray, ncomp: int = 3, cells=None) -> np.ndarray:
    """y = M u, the DG mass matrix m(v, u) = sum_K int_K v . u dx by Gauss quadrature (G1):
    y[K,c,i] = sum_q JxW_q phi_i(x_q) u_c(x_q), u_c(x_q) = sum_j u[K,c,j] phi_j(x_q).
    This is the time-derivative term (gamma_0/dt) M u of the viscous step of the projection
    scheme (BDF).  Written as the full-tensor definition;
    with the collocation basis (G2) Phi is the identity, so M is diagonal — pinned, not assumed."""
    d = disc
    nc = d.mesh.n_cells
    U = u.reshape(nc, ncomp, d.N)
    full = cells is None
    cells = np.arange(nc) if full else np.asarray(cells)
    _, JxW, _ = d.vol_geom(cells)
    uq = np.einsum("qj,kcj->kcq", d.Phi, U[cells])
    y = np.einsum("qi,kq,kcq->kci", d.Phi, JxW, uq)
    return y.reshape(-1) if full else y


def helmholtz_apply(disc: Disc, u: np.ndarray, nu, mass: float, cells=None) -> np.ndarray:
    """y = (mass M + A(nu)) u: the Helmholtz-type operator of the viscous step
    (gamma_0/dt) M + A(nu)."""
    y = viscous_apply(disc, u, nu, cells=cells)
    if mass != 0.0:
        y = y + mass * mass_apply(disc, u, 3, cells=cells)
    return y


def penalty_apply(disc: Disc, u: np.ndarray, tau_div: np.ndarray, tau_cont: np.ndarray, cells=None,
                  chunk: int = 4096) -> np.ndarray:
    """y = A_pen u, the left-hand side of the divergence/continuity penalty step
    (eqn:penalty_step), homogeneous part:
      sum_e (v, u)_e + (div v, tau_div^e div u)_e + (v.n, tau_cont [[u]].n)_{boundary of e}
    with the oriented jump [[u]] = u(e) - u(neighbour) on interior/periodic faces, [[u]] = u on
    Dirichlet faces (boundary data g_u moves to the right-hand side), nothing on Neumann faces.
    Readings (P1/P2): tau_div^e, tau_cont^e are per-cell inputs (the paper takes them
    from Fehn2018b without formulas); on an interior face the continuity weight is
    (tau_cont^- + tau_cont^+)/2 from both sides (symmetric operator), on a Dirichlet face the
    cell's own tau_cont.  Full-tensor quadrature, Gauss n_q = k+1 (G1).  Output [cell][c][i]."""
    full = cells is None
    d = disc
    nc, N = d.mesh.n_cells, d.N
    U = u.reshape(nc, 3, N)
    cells, row = _prepare(d, cells)
    y = np.zeros((len(cells), 3, N))
    for sl in _chunks(len(cells), chunk):
        cs = cells[sl]
        _, JxW, Jinv = d.vol_geom(cs)
        uq = np.einsum("qj,kcj->kcq", d.Phi, U[cs])
        y[sl] += np.einsum("qi,kq,kcq->kci", d.Phi, JxW, uq)                  # (v, u)
        G = grad_at(d, U[cs], d.dPhi, Jinv)                                    # [C,Q,3,3] du_i/dx_j
        div = np.einsum("cqii->cq", G)
        w = (tau_div[cs][:, None] * JxW) * div                                 # tau_div JxW div u
        # div v for v = e_c phi_n: d phi_n / d x_c = sum_d dPhi[d,q,n] Jinv[q,d,c]
        y[sl] += np.einsum("kq,dqn,kqdc->kcn", w, d.dPhi, Jinv)

    inter, bnd = d.unique_faces(cells)

    def add(cs, contrib):
        r = row[cs]
        m = r >= 0
        np.add.at(y, r[m], contrib[m])

    def side(cs, f, perm=None):
        _, _, n, dA = d.face_geom(cs, f)
        val = np.einsum("pn,kcn->kcp", d.PhiF[f], U[cs])                      # [C,3,P]
        Phi = d.PhiF[f]
        if perm is not None:
            val = np.take_along_axis(val, perm[:, None, :], axis=2)
            Phi_c = Phi[perm]
        else:
            Phi_c = np.broadcast_to(Phi, (len(cs),) + Phi.shape)
        return val, Phi_c, n, dA

    for (fa, fb), (a_all, b_all, perm_all) in _group_faces(d, inter).items():
        for sl in _chunks(len(a_all), chunk):
            a, b, perm = a_all[sl], b_all[sl], perm_all[sl]
            ua, Phia, n, dA = side(a, fa)
            ub, Phib, _, _ = side(b, fb, perm)
            tau = 0.5 * (tau_cont[a] + tau_cont[b])[:, None]
            jn = np.einsum("kcp,kpc->kp", ua - ub, n)                          # [[u]].n from K-
            coef = dA * tau * jn                                               # times v.n
            add(a, np.einsum("kp,kpc,kpn->kcn", coef, n, Phia))
            add(b, np.einsum("kp,kpc,kpn->kcn", -coef, n, Phib))                # v+ . n- = -(v+ . n+)
    for f in range(6):
        cs = np.array([c for (c, g, t) in bnd if g == f and t == 1], dtype=np.int64)
        if len(cs) == 0:
            continue
        ua, Phia, n, dA = side(cs, f)
        jn = np.einsum("kcp,kpc->kp", ua, n)
        add(cs, np.einsum("kp,kpc,kpn->kcn", dA * tau_cont[cs][:, None] * jn, n, Phia))
    return y.reshape(-1) if full else y


def convective_apply(disc: Disc, u: np.ndarray, w: np.ndarray, cells=None, chunk: int = 4096) -> np.ndarray:
    """y = C(w) u, the upwind DG convective term of eqn:convective_term_weak (
    SURVEY §8(f) f4), homogeneous part, linear in u for a given transport field w:
      c_h^e(v, u; w) = (v, (w.grad) u)_e - (v, ({{w}}.n) u)_{de} + (v, ({{w}}.n) u^dag)_{de},
      u^dag = {{u}} + 1/2 sign({{w}}.n) [[u]],  [[u]] = u(e) - u(neighbour),
    so the face integrand from e is ({{w}}.n)(u^dag - u) = min({{w}}.n, 0) (u(nb) - u(e)).
    Readings (F4a-F4c): the operator written \\convectiveterm{u}{w} is (w.grad)u (the
    strong/convective form the boundary terms above belong to); on Dirichlet faces the exterior
    states are the mirror states u+ = -u, w+ = -w (homogeneous data, as G7), so {{w}} = 0 there;
    on Neumann faces u+ = u, w+ = w (no jump: no term); periodic faces are interior.
    Full-tensor quadrature, Gauss n_q = k+1 (G1).  Output [cell][c][i]."""
    full = cells is None
    d = disc
    nc, N = d.mesh.n_cells, d.N
    U = u.reshape(nc, 3, N)
    Wf = w.reshape(nc, 3, N)
    cells, row = _prepare(d, cells)
    y = np.zeros((len(cells), 3, N))
    for sl in _chunks(len(cells), chunk):
        cs = cells[sl]
        _, JxW, Jinv = d.vol_geom(cs)
        G = grad_at(d, U[cs], d.dPhi, Jinv)                            # [C,Q,3,3] du_i/dx_j
        wq = np.einsum("qj,kcj->kqc", d.Phi, Wf[cs])                   # w at the points [C,Q,3]
        conv = np.einsum("kqij,kqj->kqi", G, wq)                       # (w.grad) u  [C,Q,3]
        y[sl] += np.einsum("qn,kq,kqi->kin", d.Phi, JxW, conv)

    inter, bnd = d.unique_faces(cells)

    def add(cs, contrib):
        r = row[cs]
        m = r >= 0
        np.add.at(y, r[m], contrib[m])

    def side(cs, f, perm=None):
        _, _, n, dA = d.face_geom(cs, f)
        uu = np.einsum("pn,kcn->kpc", d.PhiF[f], U[cs])
        ww = np.einsum("pn,kcn->kpc", d.PhiF[f], Wf[cs])
        Phi = d.PhiF[f]
        if perm is not None:
            uu = np.take_along_axis(uu, perm[..., None], axis=1)
            ww = np.take_along_axis(ww, perm[..., None], axis=1)
            Phi_c = Phi[perm]
        else:
            Phi_c = np.broadcast_to(Phi, (len(cs),) + Phi.shape)
        return uu, ww, Phi_c, n, dA

    for (fa, fb), (a_all, b_all, perm_all) in _group_faces(d, inter).items():
        for sl in _chunks(len(a_all), chunk):
            a, b, perm = a_all[sl], b_all[sl], perm_all[sl]
            ua, wa, Phia, n, dA = side(a, fa)
            ub, wb, Phib, _, _ = side(b, fb, perm)
            wn = np.einsum("kpc,kpc->kp", 0.5 * (wa + wb), n)           # {{w}}.n, n from K-
            # K- side: min(wn, 0) (u+ - u-);  K+ side (normal -n): min(-wn, 0) (u- - u+)
            add(a, np.einsum("kp,kpc,kpn->kcn", dA * np.minimum(wn, 0.0), ub - ua, Phia))
            add(b, np.einsum("kp,kpc,kpn->kcn", dA * np.minimum(-wn, 0.0), ua - ub, Phib))
    # boundary faces: Dirichlet ({{w}} = 0) and Neumann (no jump) contribute nothing
    return y.reshape(-1) if full else y
