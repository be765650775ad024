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


# ---------------------------------------------------------------- GLL collocation (row f2 quadrature variant)
@pytest.mark.parametrize("dim,n,p", [(2, (3, 2), 4), (3, (2, 2, 2), 3)])
def test_gll_collocation_cartesian_kronecker(dim, n, p):
    """Cartesian mesh: the GLL rule integrates the 1D stiffness integrand (degree
    2p - 2) exactly but lumps the 1D mass (degree 2p) to diag(w_i h), so collocated
    K_p = sum_j K_j (x) prod_{i != j} M^GLL_i with the exact 1D stiffness, and it
    differs from the Gauss K_p."""
    cfg = small_config("C3" if dim == 3 else "C1", n, p=p)
    V = vertices(cfg)
    Pc = O.Problem(dim, cfg.n, p, V, quad="gll")
    from numpy.polynomial import legendre as Lg
    xi = indep.gll_nodes(p)
    c = np.zeros(p + 1)
    c[p] = 1.0
    w = 1.0 / (p * (p + 1) * Lg.legval(2 * xi - 1, c) ** 2)
    Ks, Ml = [], []
    for nk in cfg.n:
        K1, _ = indep.fe_1d(p, nk)
        h = 1.0 / nk
        M = np.zeros(nk * p + 1)
        for e in range(nk):
            M[e * p:e * p + p + 1] += w * h
        Ks.append(K1)
        Ml.append(np.diag(M))
    K = indep.kron_sum(Ks, Ml)
    N = [nk * p + 1 for nk in cfg.n]
    free = ~indep.boundary_mask(N)
    v = np.random.default_rng(9).standard_normal(Pc.ndof)
    v[~free] = 0.0
    y = Pc.apply(v)
    assert np.abs(y[free] - (K @ v)[free]).max() <= 1e-12 * np.abs(K).max()
    yg = O.Problem(dim, cfg.n, p, V).apply(v)
    assert np.abs(yg[free] - y[free]).max() > 1e-6 * np.abs(y).max()


def test_gll_collocation_equals_independent_kronecker_on_perturbed():
    """Perturbed (bilinear) mesh: the collocated operator differs from Gauss, and
    equals sum_q w_q^GLL (J^{-T} grad l_a . J^{-T} grad l_b) detJ at the nodes,
    recomputed here from numpy GLL weights and the vertex array."""
    cfg = small_config("C2", (2, 2), p=3)
    V = vertices(cfg)
    Pc = O.Problem(2, cfg.n, 3, V, quad="gll")
    Pg = O.Problem(2, cfg.n, 3, V)
    xi = indep.gll_nodes(3)
    from numpy.polynomial import legendre as Lg
    c = np.zeros(4)
    c[3] = 1.0
    w = 1.0 / (3 * 4 * Lg.legval(2 * xi - 1, c) ** 2)          # GLL weights on [0,1]
    _, D = indep.lagrange_tables(xi, xi)
    nv = cfg.n[0] + 1
    Vv = V.reshape(-1, 2)
    for e in range(4):
        ex, ey = e % 2, e // 2
        corners = [Vv[(ex + a) + nv * (ey + b)] for b in (0, 1) for a in (0, 1)]
        K = np.zeros((16, 16))
        for qy in range(4):
            for qx in range(4):
                s, t = xi[qx], xi[qy]
                J = (-(1 - t) * np.outer(corners[0], [1, 0]) + (1 - t) * np.outer(corners[1], [1, 0])
                     - t * np.outer(corners[2], [1, 0]) + t * np.outer(corners[3], [1, 0])
                     - (1 - s) * np.outer(corners[0], [0, 1]) - s * np.outer(corners[1], [0, 1])
                     + (1 - s) * np.outer(corners[2], [0, 1]) + s * np.outer(corners[3], [0, 1]))
                Ji = np.linalg.inv(J)
                G = np.zeros((16, 2))
                for a in range(16):
                    ax, ay = a % 4, a // 4
                    gref = np.array([D[qx, ax] * (ay == qy), (ax == qx) * D[qy, ay]])
                    G[a] = Ji.T @ gref
                K += w[qx] * w[qy] * np.linalg.det(J) * G @ G.T
        assert np.abs(Pc.elem_matrix(e) - K).max() <= 1e-12 * np.abs(K).max()
        assert np.abs(Pg.elem_matrix(e) - K).max() > 1e-8 * np.abs(K).max()


# ---------------------------------------------------------------- RCM ordering (row f2)
def _rcm_reference(A):
    """Reading r5 written out with scipy's graph tools: BFS distances give the level
    sets every Cuthill-McKee order must respect."""
    import scipy.sparse.csgraph as cg
    return cg.shortest_path(A, unweighted=True)


def test_rcm_tridiagonal_is_reverse_path_and_exact():
    import scipy.sparse as sp
    n = 9
    T = sp.diags([-1.0, 2.1, -1.0], [-1, 0, 1], shape=(n, n)).tocsr()
    r = np.random.default_rng(4).standard_normal(n)
    order, z = O.mdf_ilu(T, ordering=2, r=r)
    assert list(order) == list(range(n - 1, -1, -1))     # BFS 0..n-1 from the min-degree end, reversed
    assert np.allclose(T @ z, r, rtol=1e-13, atol=1e-13)  # no fill on a path: ILU(0) exact


def test_rcm_visits_by_bfs_levels_and_degree():
    """On a patch-like 27-point box graph the (reversed) RCM order visits nodes in
    nondecreasing graph distance from its start, the start has minimum degree, and
    among the unvisited neighbours of each node lower degree comes first."""
    import scipy.sparse as sp
    ex, ey, ez = 5, 4, 3
    n = ex * ey * ez
    rows, cols = [], []
    for i in range(n):
        x, y, z = i % ex, (i // ex) % ey, i // (ex * ey)
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    X, Y, Z = x + dx, y + dy, z + dz
                    if 0 <= X < ex and 0 <= Y < ey and 0 <= Z < ez:
                        rows.append(i)
                        cols.append(X + ex * (Y + ey * Z))
    A = sp.csr_matrix((np.where(np.array(rows) == np.array(cols), 30.0, -1.0), (rows, cols)), shape=(n, n))
    order, _ = O.mdf_ilu(A, ordering=2)
    cm = list(order)[::-1]
    assert sorted(cm) == list(range(n))
    deg = np.diff(A.indptr) - 1
    assert deg[cm[0]] == deg.min() and cm[0] == int(np.argmin(deg))
    dist = _rcm_reference(A)[cm[0]]
    assert np.all(np.diff(dist[cm]) >= 0)


@pytest.mark.parametrize("dim,n,p", [(2, (4, 4), 4), (3, (3, 3, 3), 3)])
def test_rcm_patches_converge_like_mdf(dim, n, p):
    """MDF- and RCM-ordered ILU give comparable iteration counts."""
    cfg = small_config("C2" if dim == 2 else "C5", n, p=p)
    its = {}
    for ordering in ("mdf", "rcm"):
        P = O.Problem(dim, cfg.n, cfg.p, vertices(cfg))
        P.schwarz_setup("vertex", ordering, "gmg")
        b = P.rhs(np.ones(P.quad_points().shape[0]))
        its[ordering] = P.pcg(b, 1e-8)[1]["iters"]
    assert abs(its["rcm"] - its["mdf"]) <= 0.3 * its["mdf"], its


# ---------------------------------------------------------------- B(1): single patch, R_0 at the bottom (row f2)
def test_single_patch_b1_matches_paper_table():
    """P:785-793 / Table tab:cart-iters (golden file): the single-patch preconditioner
    B(1) = element-structured V-cycle on K_h with MDF-ILU(0) smoothing and one R_0
    V-cycle at its p = 1 bottom.  With R_0 = GMG in place of BoomerAMG (reading c11)
    the counts land within 2 iterations of the paper's (p = 2, 4, 8; n = 2, 4, 8)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "tab_cart_iters.txt")
    ref = {}
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t) for t in line.split()]
        ref[v[0]] = dict(zip([2, 4, 8, 16, 32], v[1:]))
    from workloads import rhs_function
    for p in (2, 4, 8):
        for nn in (2, 4, 8):
            cfg = small_config("C1", (nn, nn), p=p)
            P = O.Problem.from_config(cfg)
            b = P.rhs(rhs_function(cfg, P.quad_points()))
            P.schwarz_setup("single", "mdf", "gmg")
            its = P.pcg(b, 1e-8)[1]["iters"]
            assert abs(its - ref[p][nn]) <= 2, (p, nn, its, ref[p][nn])
