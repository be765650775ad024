"""Large GPU-vs-oracle parity cases (the oracle runs on the GPU box's host cores):
the thread-mode V-cycle at a size spanning several warp-slot tiles, C3 at full size,
the C4 recipe at 16^3 with its three penalties and weak boundary data, and C5 at
64^3 (slow: LORPC_SLOW=1).  north_star: preconditioner apply within
relative 1e-11, PCG iterations within +-1 and the same final residual tolerance."""
import numpy as np
import pytest

import oracle as O
from parity_util import iters_match
from workloads import (dirichlet_function, get_config, parity_vector, random_free_rhs, rhs_function,
                       small_config, vertices)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-11


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


def _cg(L, cfg, ordering="mdf"):
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
    prec = L.Prec(L.Lor(mesh), patch_kind=cfg.patch_kind, ordering=ordering)
    P = O.Problem.from_config(cfg)
    P.schwarz_setup(cfg.patch_kind, ordering, "gmg")
    return mesh, prec, P


def _pcg_check(L, mesh, prec, P, bo, tol):
    x = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    rep = L.pcg_solve(mesh, prec, dev(bo), x, tol)
    xo, ro = P.pcg(bo, tol)
    assert rep["converged"] and rep["rel_res"] <= tol
    assert iters_match(P, bo, tol, rep["iters"], ro["iters"]), (rep["iters"], ro["iters"])
    assert rel(x.cpu().numpy(), xo) <= 100 * tol
    return rep, ro


@pytest.mark.parametrize("ordering", ["mdf", "rcm"])
def test_c5_recipe_32cubed_multi_tile(L, ordering):
    """C5 recipe at 32^3 (33^3 vertex patches: two 32 x 32 warp-slot tiles per axis of
    the thread-mode V-cycle; with RCM the U-record kernels, patches grouped into warps
    by box shape): element-wise preconditioner parity and PCG."""
    cfg = small_config("C5", (32, 32, 32))
    mesh, prec, P = _cg(L, cfg, ordering)
    assert "thread-mode" in prec.kernel()
    assert ("U-records" in prec.kernel()) == (ordering == "rcm")
    r = parity_vector(P.ndof, seed=50)
    X = P.node_coords()
    free = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    r[~free] = 0.0
    z = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z)
    zo = P.precond(r)
    zg = z.cpu().numpy()
    assert rel(zg, zo) <= TOL
    assert np.abs(zg - zo).max() <= TOL * np.abs(zo).max()
    _pcg_check(L, mesh, prec, P, random_free_rhs(cfg), cfg.tol)


@pytest.mark.slow
def test_c3_full_size_pcg(L):
    """C3 at full size (32^3, p = 4, 2.1M DOFs): PCG iterations and solution (the
    oracle needs ~5 min on 16 host cores)."""
    cfg = get_config("C3")
    mesh, prec, P = _cg(L, cfg)
    bo = P.rhs(rhs_function(cfg, P.quad_points()))
    _pcg_check(L, mesh, prec, P, bo, cfg.tol)


def _c4(L, n, c):
    """C4 recipe (SIPG, p = 5, eta = (p+1)^2 c, exp-sin solution imposed weakly):
    right-hand side with the Nitsche boundary terms, PCG."""
    cfg = small_config("C4", n)
    eta = (cfg.p + 1) ** 2 * c
    V = vertices(cfg)
    mesh = L.Mesh(3, cfg.n, cfg.p, V, disc=1, eta=eta)
    prec = L.Prec(L.Lor(mesh))
    P = O.Problem(3, cfg.n, cfg.p, V, disc="sipg", eta=eta)
    P.schwarz_setup("vertex", "mdf", "gmg")
    xq = torch.empty(mesh.n_quad * 3, dtype=torch.float64, device="cuda")
    xb = torch.empty(mesh.n_bface_quad * 3, dtype=torch.float64, device="cuda")
    mesh.quad_points(xq, xb)
    Xo, Xbo = P.quad_points(), P.bface_points()
    b = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    mesh.rhs_assemble(dev(rhs_function(cfg, Xo)), dev(dirichlet_function(cfg, Xbo)), b)
    bo = P.rhs(rhs_function(cfg, Xo))
    P.rhs_bc(dirichlet_function(cfg, Xbo), bo)
    assert rel(b.cpu().numpy(), bo) <= TOL
    _pcg_check(L, mesh, prec, P, bo, cfg.tol)


@pytest.mark.parametrize("c", [1.0, 10.0, 1000.0])
def test_c4_recipe_6cubed_sipg(L, c):
    _c4(L, (6, 6, 6), c)


@pytest.mark.slow
@pytest.mark.parametrize("c", [1.0, 10.0, 1000.0])
def test_c4_recipe_16cubed_sipg(L, c):
    """16^3 (885K DG DOFs): the oracle's DG solve takes ~10 min per penalty."""
    _c4(L, (16, 16, 16), c)


@pytest.mark.slow
@pytest.mark.parametrize("ordering", ["mdf", "rcm"])
def test_c5_recipe_64cubed_pcg(L, ordering):
    """C5 recipe at 64^3 (7.2M DOFs), PCG against the oracle."""
    cfg = small_config("C5", (64, 64, 64))
    mesh, prec, P = _cg(L, cfg, ordering)
    _pcg_check(L, mesh, prec, P, random_free_rhs(cfg), cfg.tol)
