"""Q-mode fused patch V-cycle (vcycle_w.cu k_vq, kernel mode 4): LP = 2 / 4 / 8 lanes
per patch, 32 / LP patches per warp sharing one sweep schedule (structure-only
orderings: natural, RCM = reading r5, P:599 / P:606-608), the factor streamed through
a cp.async ring.  Element-wise preconditioner parity with the oracle (north_star:
relative 1e-11), agreement with the thread-mode kernels of the same ordering, PCG
iterations within +-1."""
import numpy as np
import pytest

import oracle as O
from workloads import parity_vector, random_free_rhs, rhs_function, small_config, vertices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-11

CASES = {
    "C5s": small_config("C5", (4, 3, 5)),         # 3D vertex patches, 8 box shapes, padded warps
    "C5t": small_config("C5", (9, 2, 7)),         # thin axis: only clipped shapes along y
    "C5p2": small_config("C5", (5, 4, 3), p=2),   # p = 2: 3 x 3 x 3 boxes
    "C5m": small_config("C5", (12, 11, 10)),      # several warps per shape, ragged last warps
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


@pytest.mark.parametrize("lp", [4, 2, 8])
@pytest.mark.parametrize("ordering", ["rcm", "natural"])
@pytest.mark.parametrize("name", list(CASES))
def test_qmode_precond_parity(L, name, ordering, lp, monkeypatch):
    cfg = CASES[name]
    monkeypatch.setenv("LORPC_QMODE", "1")
    monkeypatch.setenv("LORPC_QLP", str(lp))
    mesh, prec = _prec(L, cfg, ordering)
    assert "Q-mode" in prec.kernel()
    P = O.Problem.from_config(cfg)
    P.schwarz_setup(cfg.patch_kind, ordering, "gmg")
    r = _free_r(P, 61)
    z = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z)
    zo = P.precond(r)
    zg = z.cpu().numpy()
    assert np.linalg.norm(zg - zo) <= TOL * np.linalg.norm(zo)
    assert np.abs(zg - zo).max() <= TOL * np.abs(zo).max()
    # the thread-mode kernels of the same ordering
    monkeypatch.setenv("LORPC_QMODE", "0")
    mesh2, prec2 = _prec(L, cfg, ordering)
    assert "thread-mode" in prec2.kernel()
    z2 = torch.empty_like(z)
    prec2.apply(dev(r), z2)
    assert np.abs(z2.cpu().numpy() - zg).max() <= 1e-12 * np.abs(zg).max()


@pytest.mark.parametrize("name", ["C5s", "C5m"])
def test_qmode_pcg_parity(L, name, monkeypatch):
    cfg = CASES[name]
    monkeypatch.setenv("LORPC_QMODE", "1")
    mesh, prec = _prec(L, cfg, "rcm")
    assert "Q-mode" in prec.kernel()
    P = O.Problem.from_config(cfg)
    P.schwarz_setup(cfg.patch_kind, "rcm", "gmg")
    bo = random_free_rhs(cfg) if cfg.rhs == "randn" else P.rhs(rhs_function(cfg, P.quad_points()))
    x = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    rep = L.pcg_solve(mesh, prec, dev(bo), x, cfg.tol)
    xo, ro = P.pcg(bo, cfg.tol)
    assert rep["converged"] and rep["rel_res"] <= cfg.tol
    assert abs(rep["iters"] - ro["iters"]) <= 1
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 100 * cfg.tol * np.linalg.norm(xo)


def test_qmode_mdf_falls_back(L, monkeypatch):
    """MDF orderings differ from patch to patch: no shared schedule, thread mode."""
    monkeypatch.setenv("LORPC_QMODE", "1")
    mesh, prec = _prec(L, CASES["C5s"], "mdf")
    assert "thread-mode" in prec.kernel()
