"""Pins of the oracle's h-multigrid pieces, CPU only:
the h-prolongation reproduces every Q_k polynomial exactly on nested Cartesian meshes (catches
octant / orientation / index errors), the restriction is the Galerkin transpose for the mass
matrix (P^T M_fine P = M_coarse exactly, since Gauss n = k+1 integrates Q_2k exactly — catches a
wrong transpose or child sum), and the V-cycle over p- and h-levels with a direct coarse solve
is a symmetric contraction."""
import numpy as np
import pytest

from inputs import cube, cube_parent_map, uniform
from inputs.vectors import field_to_dofs, node_positions
from oracle import dense, dg, laws, mg


def _poly(x, k, comp):
    """A Q_k polynomial with all monomials of the top degree present (different per component)."""
    X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
    c = 1.0 + comp
    return (c * X ** k * Y ** max(k - 1, 0) * (Z + 0.3) ** k - 0.7 * Y ** k * Z + (comp - 1.5) * X * Y * Z
            + 0.2 * Z ** k - comp)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_h_prolongation_reproduces_polynomials(k):
    Nf = 4
    mc, mf = cube(Nf // 2), cube(Nf)
    parent, octant = cube_parent_map(Nf)
    xc, xf = node_positions(mc, k), node_positions(mf, k)
    vc = field_to_dofs(np.stack([_poly(xc, k, c) for c in range(3)], axis=-1))
    vf = field_to_dofs(np.stack([_poly(xf, k, c) for c in range(3)], axis=-1))
    out = mg.h_prolongate(vc, k, parent, octant, ncomp=3)
    assert np.abs(out - vf).max() < 1e-12 * np.abs(vf).max()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_h_restriction_is_galerkin_for_the_mass_matrix(k):
    Nf = 4
    mc, mf = cube(Nf // 2), cube(Nf)
    parent, octant = cube_parent_map(Nf)
    dc, df = dg.Disc(mc, k), dg.Disc(mf, k)
    x = uniform(0, mc.n_cells * 3 * dc.N)
    lhs = mg.h_restrict(dg.mass_apply(df, mg.h_prolongate(x, k, parent, octant, 3)), k, parent, octant,
                        mc.n_cells, 3)
    rhs = dg.mass_apply(dc, x)
    assert np.abs(lhs - rhs).max() < 1e-14 * np.abs(rhs).max() * 10
    # adjointness of the pair as stated: <R r, x> = <r, P x>
    r = uniform(1, mf.n_cells * 3 * df.N)
    assert abs(mg.h_restrict(r, k, parent, octant, mc.n_cells, 3) @ x
               - r @ mg.h_prolongate(x, k, parent, octant, 3)) < 1e-12 * np.linalg.norm(r) * np.linalg.norm(x)


def test_cph_vcycle_with_direct_coarse_solve_is_symmetric_contraction():
    """Poisson (C4 coefficient law) on cube(4): p-levels 2 -> 1, then h-level cube(2) at k = 1 solved
    directly.  V is linear and symmetric, and the error propagator I - V A has spectral radius < 1."""
    law = laws.C4_LAW
    mf, mc = cube(4), cube(2)
    parent, octant = cube_parent_map(4)
    levels = []
    for k in (2, 1):
        d = dg.Disc(mf, k)
        Ad = dense.assemble_poisson(d, dg.AnalyticNu(d, law))
        levels.append({"apply": (lambda x, Ad=Ad: Ad @ x), "Dinv": 1.0 / np.diag(Ad), "A": Ad})
    levels[0]["restrict"] = lambda r: mg.restrict(r, 2, 1, mf.n_cells)
    levels[0]["prolongate"] = lambda x: mg.prolongate(x, 2, 1, mf.n_cells)
    levels[1]["restrict"] = lambda r: mg.h_restrict(r, 1, parent, octant, mc.n_cells)
    levels[1]["prolongate"] = lambda x: mg.h_prolongate(x, 1, parent, octant)
    dcc = dg.Disc(mc, 1)
    Ac = dense.assemble_poisson(dcc, dg.AnalyticNu(dcc, law))
    levels.append({"apply": (lambda x: Ac @ x), "Dinv": 1.0 / np.diag(Ac), "solve": lambda b: np.linalg.solve(Ac, b)})
    for L in levels[:2]:
        L["lam_hi"] = 1.2 * mg.lanczos_lambda_max(L["apply"], L["Dinv"], uniform(2, len(L["Dinv"])), 20)
    A0 = levels[0]["A"]
    n = A0.shape[0]
    V = np.array([mg.vcycle(levels, e) for e in np.eye(n)]).T
    assert np.abs(V - V.T).max() < 1e-10 * np.abs(V).max()
    rho = np.abs(np.linalg.eigvals(np.eye(n) - V @ A0)).max()
    assert rho < 1.0          # 0.67 at the 1e4 coefficient contrast of C4
    # the direct coarse solve is exact: a single "solve" level returns A^-1 b
    b = uniform(0, Ac.shape[0])
    assert np.allclose(mg.vcycle([levels[-1]], b), np.linalg.solve(Ac, b), rtol=0, atol=1e-12 * np.abs(np.linalg.solve(Ac, b)).max())
