"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test checks the oracle against something other than itself: closed forms
(GLL/Gauss rules, 1D matrices), textbook identities (Kronecker structure of
Cartesian operators), brute force (dense eigenvalues,
dense solves), or statements of the paper (finite-overlap bound P:361-362,
FEM-SEM equivalence Prop. prop:fem-sem P:227-237, robustness Cor. cor:as
P:531-537).  Independent constructions live in tests/indep.py.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sl
import scipy.sparse as sp

import oracle as O
from tests import indep
from workloads import (CONFIGS, exact_solution, rhs_function, small_config, vertices,
                       dirichlet_function)

pytestmark = pytest.mark.filterwarnings("ignore")


def cart(dim, n, p):
    cfg = small_config("C1" if dim == 2 else "C3", n, p=p)
    return cfg, O.Problem.from_config(cfg)


# ---------------------------------------------------------------- basis
def test_gll_closed_forms():
    xi, w, *_ = O.basis(1)
    assert np.allclose(xi, [0, 1], atol=1e-15) and np.allclose(w, [0.5, 0.5], atol=1e-15)
    xi, w, *_ = O.basis(2)
    assert np.allclose(xi, [0, 0.5, 1], atol=1e-15) and np.allclose(w, [1 / 6, 2 / 3, 1 / 6], atol=1e-15)
    xi, w, *_ = O.basis(3)
    s = 1 / math.sqrt(5)
    assert np.allclose(xi, [0, (1 - s) / 2, (1 + s) / 2, 1], atol=1e-15)
    assert np.allclose(w, [1 / 12, 5 / 12, 5 / 12, 1 / 12], atol=1e-15)
    xi, w, *_ = O.basis(4)
    s = math.sqrt(3 / 7)
    assert np.allclose(xi, [0, (1 - s) / 2, 0.5, (1 + s) / 2, 1], atol=1e-15)
    assert np.allclose(w, [1 / 20, 49 / 180, 16 / 45, 49 / 180, 1 / 20], atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 5, 7, 12])
def test_rules_exactness_and_symmetry(p):
    xi, w, xg, wg, B, D = O.basis(p)
    assert np.allclose(xi + xi[::-1], 1.0, atol=1e-14)
    assert np.allclose(xi, indep.gll_nodes(p), atol=1e-14)
    for k in range(2 * p):          # GLL exact to degree 2p-1
        assert abs(np.dot(w, xi ** k) - 1 / (k + 1)) < 1e-14
    for k in range(2 * (p + 1)):    # Gauss q=p+1 exact to degree 2p+1
        assert abs(np.dot(wg, xg ** k) - 1 / (k + 1)) < 1e-14
    assert np.allclose(B.sum(1), 1.0, atol=1e-13)     # partition of unity
    assert np.allclose(D.sum(1), 0.0, atol=1e-11)
    Bi, Di = indep.lagrange_tables(indep.gll_nodes(p), indep.gauss(p + 1)[0])
    assert np.allclose(B, Bi, atol=1e-10) and np.allclose(D, Di, atol=1e-8)


def test_1d_matrices_closed_forms():
    for p, Mref in [(1, np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])),
                    (2, np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]) / 30)]:
        xi, w, xg, wg, B, D = O.basis(p)
        M = B.T @ np.diag(wg) @ B
        K = D.T @ np.diag(wg) @ D
        assert np.allclose(M, Mref, atol=1e-15)
        assert np.allclose(K @ np.ones(p + 1), 0, atol=1e-13)
    xi, w, xg, wg, B, D = O.basis(1)
    assert np.allclose(D.T @ np.diag(wg) @ D, [[1, -1], [-1, 1]], atol=1e-15)


def test_chains():
    # reading c3 / S:421 / SURVEY App. A
    assert O.chain(3) == [[0, 1, 2, 3], [0, 2, 3], [0, 3]]
    assert O.chain(4) == [[0, 1, 2, 3, 4], [0, 2, 4], [0, 4]]
    assert O.chain(5) == [[0, 1, 2, 3, 4, 5], [0, 2, 4, 5], [0, 4, 5], [0, 5]]
    assert O.chain(7) == [[0, 1, 2, 3, 4, 5, 6, 7], [0, 2, 4, 6, 7], [0, 4, 7], [0, 7]]
    for p in range(1, 21):
        assert len(O.chain(p)) <= math.ceil(math.log2(p)) + 1 if p > 1 else len(O.chain(p)) == 1


# ---------------------------------------------------------------- operator (eq:fem)
def test_single_element_p1_stiffness():
    # unit square, p=1: diagonal 2/3, edge neighbour -1/6, diagonal neighbour -1/3
    P = O.Problem(2, (1, 1), 1, np.array([[0, 0], [1, 0], [0, 1], [1, 1.0]]))
    K = P.elem_matrix(0)
    assert np.allclose(np.diag(K), 2 / 3, atol=1e-15)
    assert abs(K[0, 1] + 1 / 6) < 1e-15 and abs(K[0, 2] + 1 / 6) < 1e-15 and abs(K[0, 3] + 1 / 3) < 1e-15


@pytest.mark.parametrize("dim,n,p", [(2, (3, 2), 3), (2, (2, 2), 5), (3, (2, 2, 2), 2), (3, (2, 1, 2), 3)])
def test_operator_equals_kronecker_formula(dim, n, p):
    """Cartesian K_p = sum_j (x)_i G_i^j from independent 1D matrices."""
    cfg, P = cart(dim, n, p)
    A = P.assemble_dense()
    Ks, Ms = zip(*[indep.fe_1d(p, nk) for nk in cfg.n])
    Kk = indep.kron_sum(list(Ks), list(Ms))
    bd = indep.boundary_mask([nk * p + 1 for nk in cfg.n])
    Kk[bd, :] = 0
    Kk[:, bd] = 0
    Kk[bd, bd] = 1.0
    assert np.abs(A - Kk).max() <= 1e-13 * np.abs(Kk).max()


def test_operator_symmetric_nullspace_perturbed():
    cfg = small_config("C2", (3, 3), p=4)
    P = O.Problem.from_config(cfg)
    A = P.assemble_dense()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    for e in range(cfg.n_el):
        K = P.elem_matrix(e)
        assert np.abs(K.sum(1)).max() < 1e-12 * np.abs(K).max()   # K_e 1 = 0
        assert np.abs(K - K.T).max() < 1e-14 * np.abs(K).max()


def test_operator_rows_match_full_apply():
    cfg = small_config("C5", (3, 3, 3))
    P = O.Problem.from_config(cfg)
    x = np.random.default_rng(0).uniform(-1, 1, P.ndof)
    y = P.apply(x)
    rows = np.arange(0, P.ndof, 7)
    assert np.allclose(P.apply_rows(x, rows), y[rows], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("dim,p", [(2, 2), (2, 3), (3, 2)])
def test_manufactured_convergence_order(dim, p):
    """L2 error of the Galerkin solution decays at order p+1 (SURVEY pin (vii))."""
    errs, hs = [], []
    ns = [2, 4, 8] if dim == 2 else [2, 4]
    for nn in ns:
        cfg = small_config("C1" if dim == 2 else "C3", (nn,) * dim, p=p)
        P = O.Problem.from_config(cfg)
        Xq = P.quad_points()
        b = P.rhs(rhs_function(cfg, Xq))
        A = P.assemble_dense()
        u = np.linalg.solve(A, b)
        errs.append(P.l2_error(u, exact_solution(cfg, Xq)))
        hs.append(1 / nn)
    rate = math.log(errs[-2] / errs[-1]) / math.log(hs[-2] / hs[-1])
    assert rate >= p + 0.8, (errs, rate)


def test_manufactured_convergence_perturbed_c2_recipe():
    errs = []
    for nn in [4, 8, 16]:
        cfg = small_config("C2", (nn, nn), p=2)
        P = O.Problem.from_config(cfg)
        Xq = P.quad_points()
        b = P.rhs(rhs_function(cfg, Xq))
        P.schwarz_setup("vertex", "mdf", "gmg")
        x, _ = P.pcg(b, 1e-12)
        errs.append(P.l2_error(x, exact_solution(cfg, Xq)))
    assert math.log2(errs[-2] / errs[-1]) >= 2.8


def test_first_eigenvalue_tends_to_d_pi2():
    """lambda_min(K_p, M_p) -> d pi^2 on [0,1]^d (continuous first Dirichlet eigenvalue)."""
    for dim in (2, 3):
        n, p = (4, 4) if dim == 2 else (2, 4)
        cfg, P = cart(dim, (n,) * dim, p)
        A = P.assemble_dense()
        Ks, Ms = zip(*[indep.fe_1d(p, n) for _ in range(dim)])
        M = Ms[0]
        for i in range(1, dim):
            M = np.kron(Ms[i], M)
        free = ~indep.boundary_mask([n * p + 1] * dim)
        lam = sl.eigh(A[np.ix_(free, free)], M[np.ix_(free, free)], eigvals_only=True)[0]
        assert abs(lam - dim * math.pi ** 2) < 1e-4 * dim * math.pi ** 2


# ---------------------------------------------------------------- LOR
def test_lor_p1_equals_high_order():
    for dim, n in [(2, (3, 4)), (3, (2, 3, 2))]:
        cfg = small_config("C2" if dim == 2 else "C5", n, p=1)
        P = O.Problem.from_config(cfg)
        P.lor_assemble()
        A = P.assemble_dense()
        Kh = P.level_matrix(0).toarray()
        X = P.node_coords()
        free = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
        assert np.abs(A[np.ix_(free, free)] - Kh[np.ix_(free, free)]).max() < 1e-13


@pytest.mark.parametrize("dim,n,p", [(2, (3, 2), 4), (3, (2, 2, 2), 3)])
def test_lor_equals_kronecker_sum_of_p1_on_gll(dim, n, p):
    cfg, P = cart(dim, n, p)
    P.lor_assemble()
    Kh = P.level_matrix(0).toarray()
    Ks, Ms = zip(*[indep.p1_1d(indep.gll_grid_points(p, nk)) for nk in cfg.n])
    Kk = indep.kron_sum(list(Ks), list(Ms))
    assert np.abs(Kh - Kk).max() <= 1e-13 * np.abs(Kk).max()
    assert max(np.diff(P.level_matrix(0).indptr)) <= 3 ** dim   # nnz/row bounded


def test_galerkin_levels_equal_rediscretised_q1_on_coarse_gll():
    """Reading c4 / nested Q1 spaces: on Cartesian meshes P^T A P equals the Q1
    operator re-discretised on the retained GLL points."""
    for dim, n, p in [(2, (3, 2), 7), (3, (2, 2, 2), 4)]:
        cfg, P = cart(dim, n, p)
        P.lor_assemble()
        ch = O.chain(p)
        for l in range(1, len(ch)):
            Al = P.level_matrix(l).toarray()
            Ks, Ms = zip(*[indep.p1_1d(indep.gll_grid_points(p, nk, ch[l])) for nk in cfg.n])
            Kk = indep.kron_sum(list(Ks), list(Ms))
            assert np.abs(Al - Kk).max() <= 1e-12 * np.abs(Kk).max()


def test_fem_sem_equivalence_bounded():
    """Prop. prop:fem-sem: spectral equivalence constants of (K_p, K_h) bounded in p."""
    ratios = []
    for p in [2, 3, 4, 6, 8]:
        cfg, P = cart(2, (4, 4), p)
        P.lor_assemble()
        A = P.assemble_dense()
        Kh = P.level_matrix(0).toarray()
        free = ~indep.boundary_mask([4 * p + 1] * 2)
        ev = sl.eigh(A[np.ix_(free, free)], Kh[np.ix_(free, free)], eigvals_only=True)
        ratios.append(ev[-1] / ev[0])
        if p == 3:   # independent Kronecker computation gives [0.8029, 2.8226]
            Kp = indep.kron_sum(*zip(*[indep.fe_1d(3, 4)] * 2))
            Kq = indep.kron_sum(*zip(*[indep.p1_1d(indep.gll_grid_points(3, 4))] * 2))
            ev2 = sl.eigh(Kp[np.ix_(free, free)], Kq[np.ix_(free, free)], eigvals_only=True)
            assert np.allclose([ev[0], ev[-1]], [ev2[0], ev2[-1]], rtol=1e-10)
    assert max(ratios) <= 10 and ratios[-1] / ratios[-2] < 1.2


# ---------------------------------------------------------------- ILU / MDF
def _lap5(m):
    T = sp.diags([-1, 2, -1], [-1, 0, 1], shape=(m, m))
    I = sp.identity(m)
    return (sp.kron(I, T) + sp.kron(T, I)).tocsr()


def test_ilu_tridiagonal_is_exact_and_mdf_is_natural():
    rng = np.random.default_rng(3)
    n = 12
    A = sp.diags([-np.ones(n - 1), 2.5 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()
    r = rng.standard_normal(n)
    for ordering in (0, 1):
        order, z = O.mdf_ilu(A, ordering, r)
        assert np.allclose(z, np.linalg.solve(A.toarray(), r), rtol=1e-13)
        assert list(order) == list(range(n))   # all discard weights zero -> natural tie-break


def test_ilu_diagonal_matrix():
    d = np.array([2.0, 3.0, 5.0, 7.0])
    order, z = O.mdf_ilu(sp.diags(d).tocsr(), 0, np.ones(4))
    assert np.allclose(z, 1 / d, rtol=1e-15)


def test_mdf_first_pick_is_corner_brute_force():
    """on the 3x3 5-point Laplacian the first MDF pick is a corner.  Brute
    force: discarded fill of every node computed from dense Gaussian elimination."""
    A = _lap5(3)
    Ad = A.toarray()
    pattern = Ad != 0
    w = []
    for k in range(9):
        nb = [i for i in range(9) if i != k and pattern[i, k]]
        s = 0.0
        for i in nb:
            for j in nb:
                if i != j and not pattern[i, j]:
                    s += (Ad[i, k] * Ad[k, j] / Ad[k, k]) ** 2
        w.append(s)
    corners = {0, 2, 6, 8}
    wmin = min(w)
    assert {k for k in range(9) if w[k] == wmin} == corners
    order, _ = O.mdf_ilu(A, 0)
    assert order[0] == 0 and order[0] in corners
    assert sorted(order) == list(range(9))


def test_ilu_matches_dense_incomplete_elimination():
    """M = L D L^T equals dense Gaussian elimination with fill dropped outside the
    pattern, in the oracle's own order (brute force on a 5x5 9-point LOR patch)."""
    cfg, P = cart(2, (2, 2), 3)
    P.lor_assemble()
    A0 = P.level_matrix(0).toarray()
    N = 7
    idx = [i + N * j for j in range(1, 6) for i in range(1, 6)]
    A = sp.csr_matrix(A0[np.ix_(idx, idx)])
    order, _ = O.mdf_ilu(A, 0)
    n = A.shape[0]
    Ad = A.toarray()[np.ix_(order, order)]
    pat = Ad != 0
    W = Ad.copy()
    Lm = np.eye(n)
    for k in range(n):
        for i in range(k + 1, n):
            if pat[i, k]:
                Lm[i, k] = W[i, k] / W[k, k]
        for i in range(k + 1, n):
            for j in range(k + 1, n):
                if pat[i, k] and pat[k, j] and pat[i, j]:
                    W[i, j] -= W[i, k] * W[k, j] / W[k, k]
    Dm = np.diag(np.diag(W))
    M = Lm @ Dm @ Lm.T
    r = np.random.default_rng(1).standard_normal(n)
    _, z = O.mdf_ilu(A, 0, r)
    zref = np.zeros(n)
    zref[order] = np.linalg.solve(M, r[order])
    assert np.allclose(z, zref, rtol=1e-12)
    # the MDF pick was valid at every step (reading c6 validity rule)
    assert mdf_is_valid(A.toarray(), order)


def mdf_is_valid(Ad, order, band=1e-9):
    """Replay: every pick's discarded fill is within (1+band) of the minimum."""
    n = Ad.shape[0]
    pat = Ad != 0
    W = Ad.copy()
    alive = np.ones(n, dtype=bool)
    for k in order:
        ws = {}
        for c in np.nonzero(alive)[0]:
            nb = [i for i in np.nonzero(pat[:, c])[0] if i != c and alive[i]]
            s = 0.0
            for i in nb:
                for j in nb:
                    if i != j and not pat[i, j]:
                        s += (W[i, c] * W[c, j] / W[c, c]) ** 2
            ws[c] = s
        if ws[k] > (1 + band) * min(ws.values()) + 1e-300:
            return False
        nb = [i for i in np.nonzero(pat[:, k])[0] if i != k and alive[i]]
        for i in nb:
            for j in nb:
                if pat[i, j]:
                    W[i, j] -= W[i, k] * W[k, j] / W[k, k]
        alive[k] = False
    return True


def test_mdf_validity_on_perturbed_patch():
    cfg = small_config("C2", (2, 2), p=3)
    P = O.Problem.from_config(cfg)
    P.lor_assemble()
    A0 = P.level_matrix(0).toarray()
    N = 7
    idx = [i + N * j for j in range(1, 6) for i in range(1, 6)]
    A = A0[np.ix_(idx, idx)]
    order, _ = O.mdf_ilu(sp.csr_matrix(A), 0)
    assert mdf_is_valid(A, order)


# ---------------------------------------------------------------- Schwarz (eq:as)
def dense_B(P, free):
    N = P.ndof
    B = np.zeros((N, N))
    for j in np.nonzero(free)[0]:
        e = np.zeros(N)
        e[j] = 1
        B[:, j] = P.precond(e)
    return B[np.ix_(free, free)]


@pytest.mark.parametrize("kind,bound", [("vertex", 4 + 1), ("star", 9 + 1)])
def test_schwarz_exact_solvers_finite_overlap_bound(kind, bound):
    """lambda_max(B K_h) <= (max patches covering a point) + 1 = 2^d+1 (vertex) or
    3^d+1 (star) with exact local and coarse solvers."""
    cfg, P = cart(2, (4, 4), 3)
    P.schwarz_setup(kind, "mdf", "exact", local_exact=True)
    Kh = P.level_matrix(0).toarray()
    free = ~indep.boundary_mask([13, 13])
    B = dense_B(P, free)
    ev = np.sort(np.real(np.linalg.eigvals(B @ Kh[np.ix_(free, free)])))
    assert ev[0] > 0 and ev[-1] <= bound + 1e-10
    assert abs(ev[-1] - (4.0 if kind == "vertex" else 9.0)) < 1e-8  # dense value


def test_single_patch_exact_solver_is_inverse():
    cfg, P = cart(2, (3, 3), 2)
    P.schwarz_setup("single", "mdf", "none", local_exact=True)
    Kh = P.level_matrix(0).toarray()
    free = ~indep.boundary_mask([7, 7])
    B = dense_B(P, free)
    assert np.allclose(B, np.linalg.inv(Kh[np.ix_(free, free)]), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("dim,n,p,kind", [(2, (4, 4), 3, "star"), (2, (3, 3), 4, "vertex"),
                                          (3, (2, 2, 2), 3, "vertex")])
def test_schwarz_symmetric_positive_definite(dim, n, p, kind):
    cfg = small_config("C2" if dim == 2 else "C5", n, p=p)
    P = O.Problem.from_config(cfg)
    P.schwarz_setup(kind, "mdf", "gmg")
    X = P.node_coords()
    free = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    B = dense_B(P, free)
    assert np.abs(B - B.T).max() <= 1e-13 * np.abs(B).max()
    assert np.linalg.eigvalsh(0.5 * (B + B.T))[0] > 0


def test_patch_vcycle_nearly_exact_on_cartesian_interior_patch():
    """Readings c3-c8 on a Cartesian interior vertex patch: kappa(B_mg A_j) <= 1.05
    (SURVEY App. A dense probe); here via a single-vertex patch problem: the
    middle vertex patch of a 2x2 mesh with the coarse term removed."""
    for dim, p in [(2, 3), (2, 7), (3, 3)]:
        cfg, P = cart(dim, (2,) * dim, p)
        P.schwarz_setup("vertex", "mdf", "none")
        Kh = P.level_matrix(0).toarray()
        free = ~indep.boundary_mask([2 * p + 1] * dim)
        # only the centre patch covers interior-of-domain nodes away from others:
        # isolate it: r supported on its free nodes; compare with the exact local solve
        N = 2 * p + 1
        coords = np.stack(np.meshgrid(*[np.arange(N)] * dim, indexing="ij"), -1).reshape(-1, dim)[:, ::-1]
        mid = np.all((coords > 0) & (coords < N - 1), axis=1)
        Aj = Kh[np.ix_(mid, mid)]
        # B restricted to the patch nodes equals R_centre + (other patches) ; use the
        # dedicated single-patch problem instead: 'single' on a 2x2 mesh = the centre patch
        P2 = O.Problem.from_config(cfg)
        P2.schwarz_setup("single", "mdf", "none")
        B = dense_B(P2, free)
        ev = np.sort(np.real(np.linalg.eigvals(B @ Kh[np.ix_(free, free)])))
        assert ev[-1] / ev[0] <= 1.05, (dim, p, ev[0], ev[-1])
        assert np.abs(B - B.T).max() <= 1e-14 * np.abs(B).max() * 10
        assert Aj.shape[0] == (2 * p - 1) ** dim


# ---------------------------------------------------------------- PCG
def test_pcg_p1_exact_preconditioner_one_iteration():
    cfg, P = cart(2, (4, 4), 1)
    Xq = P.quad_points()
    b = P.rhs(rhs_function(cfg, Xq))
    P.schwarz_setup("single", "mdf", "none", local_exact=True)
    x, rep = P.pcg(b, 1e-10)
    assert rep["iters"] == 1


def test_pcg_solution_matches_dense_solve_and_kappa():
    cfg = small_config("C2", (4, 4), p=3)
    P = O.Problem.from_config(cfg)
    Xq = P.quad_points()
    b = P.rhs(rhs_function(cfg, Xq))
    A = P.assemble_dense()
    P.schwarz_setup("vertex", "mdf", "gmg")
    x, rep = P.pcg(b, 1e-12)
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-9 * np.linalg.norm(xd)
    free = np.abs(np.diag(A) - 1) > 0  # Dirichlet rows are identity rows
    X = P.node_coords()
    free = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    B = dense_B(P, free)
    ev = np.sort(np.real(np.linalg.eigvals(B @ A[np.ix_(free, free)])))
    kl = O.lanczos_kappa(rep["alpha"], rep["beta"])
    assert abs(kl - ev[-1] / ev[0]) <= 0.05 * ev[-1] / ev[0]


def test_pcg_scaling_invariance():
    cfg = small_config("C2", (4, 4), p=3)
    P = O.Problem.from_config(cfg)
    b = P.rhs(rhs_function(cfg, P.quad_points()))
    P.schwarz_setup("vertex", "mdf", "gmg")
    _, r1 = P.pcg(b, 1e-10)
    _, r2 = P.pcg(1e3 * b, 1e-10)
    assert r1["iters"] == r2["iters"]


def test_kappa_bounded_in_h_and_p_2d():
    """Cor. cor:as: kappa(B K_p) bounded as h and p vary (2D, vertex patches)."""
    ks = {}
    for n in [4, 8, 16]:
        for p in [3, 5]:
            cfg = small_config("C1", (n, n), p=p)
            P = O.Problem.from_config(cfg)
            b = P.rhs(rhs_function(cfg, P.quad_points()))
            P.schwarz_setup("vertex", "mdf", "exact")
            _, rep = P.pcg(b, 1e-10)
            ks[(n, p)] = O.lanczos_kappa(rep["alpha"], rep["beta"])
    for p in [3, 5]:
        assert ks[(16, p)] / ks[(8, p)] <= 1.25
    assert max(ks.values()) < 30


# ---------------------------------------------------------------- SIPG (eq:ip)
def _dg_problem(dim, n, p, c):
    cfg = small_config("C4", n, p=p)
    if dim == 2:
        from dataclasses import replace
        cfg = replace(cfg, dim=2)
    eta = (p + 1) ** 2 * c
    return cfg, O.Problem.from_config(cfg, eta=eta)


def _dg_perm(n, p):
    """element-major (e, a) index -> Kronecker x-fastest index of the 1D DG grids."""
    nl1 = p + 1
    dim = len(n)
    perm = []
    for ez in range(n[2] if dim == 3 else 1):
        for ey in range(n[1]):
            for ex in range(n[0]):
                for az in range(nl1 if dim == 3 else 1):
                    for ay in range(nl1):
                        for ax in range(nl1):
                            ix = ex * nl1 + ax
                            iy = ey * nl1 + ay
                            iz = ez * nl1 + az
                            perm.append(ix + n[0] * nl1 * (iy + n[1] * nl1 * iz))
    return np.array(perm)


@pytest.mark.parametrize("c", [1.0, 1000.0])
def test_sipg_equals_kronecker_of_1d_sipg(c):
    """Cartesian SIPG = A1 (x) M (x) M + ... with 1D SIPG A1 and DG mass M."""
    n, p = (2, 3, 2), 2
    cfg, P = _dg_problem(3, n, p, c)
    A = P.assemble_dense()
    sig = (p + 1) ** 2 * c
    mats = [indep.sipg_1d(p, nk, sig) for nk in n]
    Ak = indep.kron_sum([m[0] for m in mats], [m[1] for m in mats])
    perm = _dg_perm(n, p)
    Ak = Ak[np.ix_(perm, perm)]
    assert np.abs(A - Ak).max() <= max(1e-14, 1e-15 * c * (p + 1) ** 2) * np.abs(Ak).max() * 10


def test_sipg_consistency_with_cg_and_penalty_monotone():
    n, p = (2, 2, 2), 2
    cfg, P = _dg_problem(3, n, p, 1.0)
    A = P.assemble_dense()
    Pc = O.Problem(3, n, p, vertices(cfg))
    K = Pc.assemble_dense()
    Xc = Pc.node_coords()
    free = np.all((Xc > 1e-12) & (Xc < 1 - 1e-12), axis=1)
    # E: CG node -> DG copies
    nl = (p + 1) ** 3
    E = np.zeros((cfg.n_el * nl, Pc.ndof))
    N = n[0] * p + 1
    for e in range(cfg.n_el):
        ex, ey, ez = e % n[0], (e // n[0]) % n[1], e // (n[0] * n[1])
        for a in range(nl):
            ax, ay, az = a % (p + 1), (a // (p + 1)) % (p + 1), a // (p + 1) ** 2
            g = (ex * p + ax) + N * ((ey * p + ay) + N * (ez * p + az))
            E[e * nl + a, g] = 1
    Ef = E[:, free]
    assert np.abs(Ef.T @ A @ Ef - K[np.ix_(free, free)]).max() < 1e-12 * np.abs(K).max()
    cfg2, P2 = _dg_problem(3, n, p, 2.0)
    D = P2.assemble_dense() - A
    assert np.linalg.eigvalsh(0.5 * (D + D.T))[0] > -1e-10 * np.abs(D).max()
    assert np.abs(A - A.T).max() < 1e-12 * np.abs(A).max()


def test_sipg_diagonal_matches_dense():
    n, p = (2, 2, 2), 2
    cfg, P = _dg_problem(3, n, p, 10.0)
    A = P.assemble_dense()
    P.schwarz_setup("vertex", "mdf", "gmg")
    assert np.allclose(P.dg_diag(), np.diag(A), rtol=1e-12)


def test_sipg_manufactured_order_weak_dirichlet():
    errs = []
    p = 2
    for nn in [3, 6]:
        cfg, P = _dg_problem(3, (nn,) * 3, p, 10.0)
        Xq = P.quad_points()
        b = P.rhs(rhs_function(cfg, Xq))
        P.rhs_bc(dirichlet_function(cfg, P.bface_points()), b)
        P.schwarz_setup("vertex", "mdf", "gmg")
        u, _ = P.pcg(b, 1e-12)
        errs.append(P.l2_error(u, exact_solution(cfg, Xq)))
    assert math.log2(errs[0] / errs[1]) >= p + 0.8


def test_dg_preconditioner_penalty_robust():
    """Thm (Antonietti): kappa(B_DG A_IP) bounded independently of eta."""
    ks = []
    for c in [1.0, 10.0, 100.0, 1000.0, 10000.0]:
        cfg, P = _dg_problem(3, (2, 2, 2), 2, c)
        b = P.rhs(rhs_function(cfg, P.quad_points()))
        P.rhs_bc(dirichlet_function(cfg, P.bface_points()), b)
        P.schwarz_setup("vertex", "mdf", "gmg")
        _, rep = P.pcg(b, 1e-10)
        ks.append(O.lanczos_kappa(rep["alpha"], rep["beta"]))
    assert max(ks) / min(ks) <= 2.0, ks


# ---------------------------------------------------------------- paper tables (golden)
def _golden(name):
    import os
    rows = {}
    path = os.path.join(os.path.dirname(__file__), "golden", name)
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t) for t in line.split()]
        rows[v[0]] = dict(zip([2, 4, 8, 16, 32], v[1:]))
    return rows


@pytest.mark.parametrize("table,kind", [("tab_cart_iters.txt", "single"),
                                        ("tab_cart_iters_patch.txt", "vertex")])
def test_iteration_counts_near_paper_tables(table, kind):
    """PCG iterations to a 1e8 reduction stay within [0.5, 1.5] x the paper's counts
    (P:811-851).  Our coarse solve is exact instead of one BoomerAMG V-cycle (c11),
    so only a band is asserted, as SPEC's acceptance 4-5 does."""
    ref = _golden(table)
    for p in [2, 4, 8]:
        for n in [2, 4, 8]:
            cfg = small_config("C1", (n, n), p=p)
            P = O.Problem.from_config(cfg)
            b = P.rhs(rhs_function(cfg, P.quad_points()))
            P.schwarz_setup(kind, "mdf", "exact")
            _, rep = P.pcg(b, 1e-8)
            assert 0.5 * ref[p][n] <= rep["iters"] <= 1.5 * ref[p][n], (p, n, rep["iters"], ref[p][n])
