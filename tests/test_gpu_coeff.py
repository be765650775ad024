"""GPU-vs-oracle parity for variable coefficients (row f3; P:881-901,
sec:variable-coeff, b1..b4): operator, preconditioner (LOR K_h with the sampled
coefficient, its Galerkin levels, patch factors and R_0), PCG.  Each side evaluates
the workloads/ coefficient at its own quadrature / subcell points."""
import numpy as np
import pytest

import oracle as O
from parity_util import iters_match
from workloads import coefficient_samples, parity_vector, small_config, vertices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-11

CASES = {"2D": small_config("C2", (6, 5), p=4), "3D": small_config("C5", (3, 2, 3), p=3)}


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1908_07071_b200 import lorpc
    return lorpc


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def both(L, cfg, kind):
    V = vertices(cfg)
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, V)
    xq = torch.empty(mesh.n_quad * cfg.dim, dtype=torch.float64, device="cuda")
    mesh.quad_points(xq)
    ns = mesh.subcell_points()
    xs = torch.empty(ns * (1 << cfg.dim) * cfg.dim, dtype=torch.float64, device="cuda")
    mesh.subcell_points(xs)
    bq, bs = coefficient_samples(kind, cfg, xq.cpu().numpy().reshape(-1, cfg.dim),
                                 xs.cpu().numpy().reshape(-1, cfg.dim))
    mesh.set_coefficient(dev(bq), dev(bs))
    P = O.Problem(cfg.dim, cfg.n, cfg.p, V)
    bqo, bso = coefficient_samples(kind, cfg, P.quad_points(), P.subcell_points())
    P.set_coefficient(bqo, bso)
    assert np.abs(xs.cpu().numpy().reshape(-1, cfg.dim) - P.subcell_points()).max() < 1e-14
    return mesh, P


@pytest.mark.parametrize("kind", ["b1", "b2", "b3", "b4"])
@pytest.mark.parametrize("case", list(CASES))
def test_coefficient_operator_precond_pcg(L, case, kind):
    cfg = CASES[case]
    mesh, P = both(L, cfg, kind)
    x = parity_vector(P.ndof, seed=51)
    y = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    mesh.apply(dev(x), y)
    yo = P.apply(x)
    assert rel(y.cpu().numpy(), yo) <= TOL
    assert np.abs(y.cpu().numpy() - yo).max() <= TOL * np.abs(yo).max()
    prec = L.Prec(L.Lor(mesh))
    P.schwarz_setup("vertex", "mdf", "gmg")
    r = parity_vector(P.ndof, seed=52)
    X = P.node_coords()
    r[~np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)] = 0.0
    z = torch.empty_like(y)
    prec.apply(dev(r), z)
    zo = P.precond(r)
    assert rel(z.cpu().numpy(), zo) <= TOL
    assert np.abs(z.cpu().numpy() - zo).max() <= TOL * np.abs(zo).max()
    bo = P.rhs(np.ones(P.quad_points().shape[0]))   # f = 1
    xg = torch.empty_like(y)
    rep = L.pcg_solve(mesh, prec, dev(bo), xg, 1e-10)
    xo, ro = P.pcg(bo, 1e-10)
    assert iters_match(P, bo, 1e-10, rep["iters"], ro["iters"]), (rep["iters"], ro["iters"])
    assert rel(xg.cpu().numpy(), xo) <= 1e-8


def test_coefficient_rejects_nonpositive_and_dg(L):
    cfg = CASES["2D"]
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
    bq = torch.ones(mesh.n_quad, dtype=torch.float64, device="cuda")
    bq[3] = 0.0
    with pytest.raises(L.LorpcError):
        mesh.set_coefficient(bq, None)
    c4 = small_config("C4", (2, 2, 2), p=2)
    dg = L.Mesh(3, c4.n, c4.p, vertices(c4), disc=1, eta=90.0)
    with pytest.raises(L.LorpcError):
        dg.set_coefficient(torch.ones(dg.n_quad, dtype=torch.float64, device="cuda"), None)


# ---------------------------------------------------------------- GLL collocation (row f2 quadrature variant)
@pytest.mark.parametrize("cfg", [small_config("C2", (5, 4), p=5), small_config("C5", (3, 2, 2), p=3)],
                         ids=["2D", "3D"])
def test_gll_collocation_parity(L, cfg):
    """quad = 1: K_p and the load vector with the (p+1)-point GLL rule; operator and
    PCG against the oracle's collocated operator."""
    V = vertices(cfg)
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, V, quad=1)
    P = O.Problem(cfg.dim, cfg.n, cfg.p, V, quad="gll")
    x = parity_vector(P.ndof, seed=53)
    y = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    mesh.apply(dev(x), y)
    yo = P.apply(x)
    assert rel(y.cpu().numpy(), yo) <= TOL
    assert np.abs(y.cpu().numpy() - yo).max() <= TOL * np.abs(yo).max()
    xq = torch.empty(mesh.n_quad * cfg.dim, dtype=torch.float64, device="cuda")
    mesh.quad_points(xq)
    assert np.abs(xq.cpu().numpy().reshape(-1, cfg.dim) - P.quad_points()).max() < 1e-14
    b = torch.empty_like(y)
    mesh.rhs_assemble(torch.ones(mesh.n_quad, dtype=torch.float64, device="cuda"), None, b)
    bo = P.rhs(np.ones(mesh.n_quad))
    assert rel(b.cpu().numpy(), bo) <= TOL
    prec = L.Prec(L.Lor(mesh))
    P.schwarz_setup("vertex", "mdf", "gmg")
    xg = torch.empty_like(y)
    rep = L.pcg_solve(mesh, prec, dev(bo), xg, 1e-10)
    xo, ro = P.pcg(bo, 1e-10)
    assert iters_match(P, bo, 1e-10, rep["iters"], ro["iters"]), (rep["iters"], ro["iters"])
    assert rel(xg.cpu().numpy(), xo) <= 1e-8


def test_gll_collocation_rejects_dg(L):
    c4 = small_config("C4", (2, 2, 2), p=2)
    with pytest.raises(L.LorpcError):
        L.Mesh(3, c4.n, c4.p, vertices(c4), disc=1, eta=90.0, quad=1)


# ---------------------------------------------------------------- B(1) single patch (row f2)
@pytest.mark.parametrize("ordering", ["mdf", "rcm"])
@pytest.mark.parametrize("cfg", [small_config("C1", (4, 4), p=3), small_config("C2", (6, 5), p=5),
                                 small_config("C5", (3, 2, 3), p=3)], ids=["2Dcart", "2Dpert", "3Dpert"])
def test_single_patch_b1_parity(L, cfg, ordering):
    """B(1): one element-structured V-cycle on the whole LOR problem, ILU(0)
    smoothing per level, R_0 at the p = 1 bottom.  Preconditioner element-wise and PCG
    against the oracle's single patch kind."""
    V = vertices(cfg)
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, V)
    prec = L.Prec(L.Lor(mesh), patch_kind="single", ordering=ordering)
    P = O.Problem(cfg.dim, cfg.n, cfg.p, V)
    P.schwarz_setup("single", ordering, "gmg")
    r = parity_vector(P.ndof, seed=55)
    X = P.node_coords()
    r[~np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)] = 0.0
    z = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z)
    zo = P.precond(r)
    assert rel(z.cpu().numpy(), zo) <= TOL
    assert np.abs(z.cpu().numpy() - zo).max() <= TOL * np.abs(zo).max()
    bo = P.rhs(np.ones(P.quad_points().shape[0]))
    x = torch.empty_like(z)
    rep = L.pcg_solve(mesh, prec, dev(bo), x, 1e-10)
    xo, ro = P.pcg(bo, 1e-10)
    assert iters_match(P, bo, 1e-10, rep["iters"], ro["iters"]), (rep["iters"], ro["iters"])
    assert rel(x.cpu().numpy(), xo) <= 1e-8
