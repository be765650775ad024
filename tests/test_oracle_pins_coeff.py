"""Pins of the oracle's variable-coefficient operators (row f3; P:881-901,
sec:variable-coeff: -div(b grad u) with b1..b4).  CPU only.

Independent of the oracle: the Kronecker constructions in tests/indep.py with
weights integrated by a higher-order Gauss rule, element scaling, and the
manufactured-solution order of convergence with a non-constant coefficient."""
import math

import numpy as np
import pytest
import scipy.linalg as sl

import indep
import oracle as O
from workloads import coefficient_b4, coefficient_samples, small_config, vertices


def cart(dim, n, p):
    cfg = small_config("C3" if dim == 3 else "C1", n, p=p)
    return cfg, O.Problem(dim, cfg.n, cfg.p, vertices(cfg))


def lin_b(X):
    return 1.0 + 3.0 * X[:, 0]      # linear in x: q = p+1 Gauss / 2-point subcell Gauss are exact


@pytest.mark.parametrize("dim,n,p", [(2, (3, 2), 3), (2, (2, 3), 5), (3, (2, 2, 2), 2)])
def test_variable_kp_equals_weighted_kronecker(dim, n, p):
    """b = 1 + 3x on a Cartesian mesh: K_p(b) = Kx(b) (x) My (x) Mz + Mx(b) (x) Ky (x) Mz + ...
    with the 1D weighted matrices integrated independently (q = p+4 Gauss)."""
    cfg, P = cart(dim, n, p)
    P.set_coefficient(lin_b(P.quad_points()), lin_b(P.subcell_points()))
    Kx, Mx = indep.fe_1d_weighted(p, cfg.n[0], lambda x: 1.0 + 3.0 * x)
    Ks, Ms = zip(*[indep.fe_1d(p, nk) for nk in cfg.n])
    K = indep.kron_sum([Kx] + list(Ks[1:]), [Mx] + list(Ms[1:]))
    N = [nk * p + 1 for nk in cfg.n]
    free = ~indep.boundary_mask(N)
    rng = np.random.default_rng(5)
    for _ in range(3):
        v = rng.standard_normal(P.ndof)
        v[~free] = 0.0
        y = P.apply(v)
        assert np.abs(y[free] - (K @ v)[free]).max() <= 1e-12 * np.abs(K).max()


@pytest.mark.parametrize("dim,n,p", [(2, (3, 2), 4), (3, (2, 2, 2), 3)])
def test_variable_kh_equals_weighted_p1_kronecker(dim, n, p):
    """K_h with b = 1 + 3x sampled at the subcell Gauss points equals the weighted Q1
    Kronecker sum on the GLL grid (the 2-point rule is exact for this integrand)."""
    cfg, P = cart(dim, n, p)
    P.set_coefficient(lin_b(P.quad_points()), lin_b(P.subcell_points()))
    P.lor_assemble()
    Kh = P.level_matrix(0).toarray()
    pts = [indep.gll_grid_points(p, nk) for nk in cfg.n]
    Kx, Mx = indep.p1_1d_weighted(pts[0], lambda x: 1.0 + 3.0 * x)
    Ks, Ms = zip(*[indep.p1_1d(pk) for pk in pts])
    K = indep.kron_sum([Kx] + list(Ks[1:]), [Mx] + list(Ms[1:]))
    assert np.abs(Kh - K).max() <= 1e-13 * np.abs(K).max()


def test_piecewise_constant_b4_scales_each_element():
    """b4 (10 or 1 per element): every element matrix is b_e times the unit one, on a
    perturbed mesh (element ordering and quadrature-point layout of the samples)."""
    cfg = small_config("C2", (4, 3), p=3)
    V = vertices(cfg)
    P1 = O.Problem(2, cfg.n, cfg.p, V)
    Pb = O.Problem(2, cfg.n, cfg.p, V)
    bq, bs = coefficient_samples("b4", cfg, Pb.quad_points(), Pb.subcell_points())
    Pb.set_coefficient(bq, bs)
    be = coefficient_b4(cfg.n_el)
    assert set(np.unique(be)) <= {1.0, 10.0}
    for e in range(cfg.n_el):
        assert np.allclose(Pb.elem_matrix(e), be[e] * P1.elem_matrix(e), rtol=1e-14, atol=1e-14)
    # K_h: each subcell scaled by its element's value, so a uniform b4 = c is c K_h
    P1.lor_assemble()
    Pc = O.Problem(2, cfg.n, cfg.p, V)
    Pc.set_coefficient(np.full(bq.shape, 10.0), np.full(bs.shape, 10.0))
    Pc.lor_assemble()
    assert np.abs(Pc.level_matrix(0).toarray() - 10.0 * P1.level_matrix(0).toarray()).max() < 1e-11


def test_variable_coefficient_manufactured_order():
    """-div(b2 grad u) = f with u = sin(pi x) sin(pi y), b2 = 100 x'^2 + y'^2 + 1,
    x' = 2x - 1: the L2 error of the Galerkin solution decays at order >= p + 0.8."""
    pi = math.pi

    def f(X):
        x, y = X[:, 0], X[:, 1]
        xp, yp = 2 * x - 1, 2 * y - 1
        b = 100 * xp ** 2 + yp ** 2 + 1
        ux, uy = pi * np.cos(pi * x) * np.sin(pi * y), pi * np.sin(pi * x) * np.cos(pi * y)
        return 2 * pi * pi * b * np.sin(pi * x) * np.sin(pi * y) - (400 * xp * ux + 4 * yp * uy)

    def u(X):
        return np.sin(pi * X[:, 0]) * np.sin(pi * X[:, 1])

    p, errs = 3, []
    for nn in (4, 8):
        cfg = small_config("C1", (nn, nn), p=p)
        P = O.Problem(2, cfg.n, p, vertices(cfg))
        from workloads import coefficient_function
        P.set_coefficient(coefficient_function("b2", P.quad_points()),
                          coefficient_function("b2", P.subcell_points()))
        A = P.assemble_dense()
        b = P.rhs(f(P.quad_points()))
        N = nn * p + 1
        free = ~indep.boundary_mask([N, N])
        x = np.zeros(P.ndof)
        x[free] = sl.solve(A[np.ix_(free, free)], b[free], assume_a="pos")
        errs.append(P.l2_error(x, u(P.quad_points())))
    assert math.log2(errs[0] / errs[1]) >= p + 0.8, errs


@pytest.mark.parametrize("kind", ["b1", "b2", "b3", "b4"])
def test_variable_coefficient_pcg_bounded(kind):
    """The LOR Schwarz preconditioner stays effective for all four coefficients
    ("The iteration counts remain bounded for all coefficients"): PCG on the
    C2 recipe (perturbed quads) at 6x6 and 12x12, p = 4, within 1.6x of each other."""
    its = []
    for nn in (6, 12):
        cfg = small_config("C2", (nn, nn), p=4)
        P = O.Problem(2, cfg.n, cfg.p, vertices(cfg))
        bq, bs = coefficient_samples(kind, cfg, P.quad_points(), P.subcell_points())
        P.set_coefficient(bq, bs)
        P.schwarz_setup("vertex", "mdf", "gmg")
        b = P.rhs(np.ones(P.quad_points().shape[0]))
        _, rep = P.pcg(b, 1e-8)
        its.append(rep["iters"])
    assert its[1] <= 1.6 * its[0] and its[1] < 200, its
