"""U-record thread-mode V-cycle (vcycle_t.cu, kernel mode 3): with a structure-only
ordering (natural; RCM = reading r5, P:599 / P:606-608) every patch of one box
shape has the same elimination order and factor sparsity, so a warp's 32 patches
share one sweep schedule and the record holds only factor values per lane.
Element-wise preconditioner parity with the oracle (north_star: relative 1e-11),
agreement with the T-record kernels of the same ordering (LORPC_UMODE=0) and PCG
iterations within +-1."""
import numpy as np
import pytest

import oracle as O
from workloads import parity_vector, random_free_rhs, rhs_function, small_config, get_config, vertices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-11

CASES = {
    "C1": get_config("C1"),                       # 2D element-star patches, p = 3
    "C5s": small_config("C5", (4, 3, 5)),         # 3D vertex patches, 8 box shapes, padded warps
    "C5t": small_config("C5", (9, 2, 7)),         # thin axis: only clipped shapes along y
    "C5p2": small_config("C5", (5, 4, 3), p=2),   # p = 2: 3 x 3 x 3 boxes
}


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1908_07071_b200 import lorpc
    return lorpc


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _free_r(P, seed):
    r = parity_vector(P.ndof, seed=seed)
    X = P.node_coords()
    free = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    r[~free] = 0.0
    return r


def _prec(L, cfg, ordering):
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
    prec = L.Prec(L.Lor(mesh), patch_kind=cfg.patch_kind, ordering=ordering)
    return mesh, prec


@pytest.mark.parametrize("ordering", ["rcm", "natural"])
@pytest.mark.parametrize("name", list(CASES))
def test_umode_precond_parity(L, name, ordering, monkeypatch):
    cfg = CASES[name]
    mesh, prec = _prec(L, cfg, ordering)
    if "thread-mode" not in prec.kernel():
        pytest.skip("configuration runs another V-cycle kernel")
    assert "U-records" in prec.kernel()
    P = O.Problem.from_config(cfg)
    P.schwarz_setup(cfg.patch_kind, ordering, "gmg")
    r = _free_r(P, 61)
    z = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z)
    zo = P.precond(r)
    zg = z.cpu().numpy()
    assert np.linalg.norm(zg - zo) <= TOL * np.linalg.norm(zo)
    assert np.abs(zg - zo).max() <= TOL * np.abs(zo).max()
    # the T-record kernels of the same ordering: the same arithmetic per patch, the
    # scatter atomics in another slot order
    monkeypatch.setenv("LORPC_UMODE", "0")
    mesh2, prec2 = _prec(L, cfg, ordering)
    assert "thread-mode" in prec2.kernel() and "U-records" not in prec2.kernel()
    z2 = torch.empty_like(z)
    prec2.apply(dev(r), z2)
    assert np.abs(z2.cpu().numpy() - zg).max() <= 1e-13 * np.abs(zg).max()


@pytest.mark.parametrize("name", ["C1", "C5s", "C5t"])
def test_umode_pcg_parity(L, name):
    cfg = CASES[name]
    mesh, prec = _prec(L, cfg, "rcm")
    P = O.Problem.from_config(cfg)
    P.schwarz_setup(cfg.patch_kind, "rcm", "gmg")
    bo = random_free_rhs(cfg) if cfg.rhs == "randn" else P.rhs(rhs_function(cfg, P.quad_points()))
    x = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    rep = L.pcg_solve(mesh, prec, dev(bo), x, cfg.tol)
    xo, ro = P.pcg(bo, cfg.tol)
    assert rep["converged"] and rep["rel_res"] <= cfg.tol
    assert abs(rep["iters"] - ro["iters"]) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 100 * cfg.tol * np.linalg.norm(xo)


def test_mdf_keeps_t_records(L):
    """MDF orderings differ from patch to patch: T-records (per-lane schedules)."""
    mesh, prec = _prec(L, CASES["C5s"], "mdf")
    assert "thread-mode" in prec.kernel() and "U-records" not in prec.kernel()
