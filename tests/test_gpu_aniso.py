"""Row f4 on the GPU (sec:aniso P:1107-1151): anisotropic strip meshes with vertex
patches extended for isotropic overlap (reading r6).  Preconditioner and PCG parity
with the oracle; iteration counts independent of the aspect ratio."""
import numpy as np
import pytest

import oracle as O
from parity_util import iters_match
from workloads import parity_vector, strip_vertices

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


@pytest.mark.parametrize("p", [3, 7])
def test_strip_extended_patches_parity(L, p):
    n = 8
    its = []
    for aspect in (1.5, 15.0, 150.0, 1500.0):
        V = strip_vertices(n, aspect)
        mesh = L.Mesh(2, (n, n), p, V)
        prec = L.Prec(L.Lor(mesh), extend=True)
        P = O.Problem(2, (n, n), p, V)
        P.schwarz_setup("vertex", "mdf", "gmg", extend=True)
        r = parity_vector(P.ndof, seed=54)
        X = P.node_coords()
        r[~np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)] = 0.0
        z = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
        prec.apply(dev(r), z)
        zo = P.precond(r)
        assert rel(z.cpu().numpy(), zo) <= TOL
        assert np.abs(z.cpu().numpy() - zo).max() <= TOL * np.abs(zo).max()
        bo = P.rhs(np.ones(P.quad_points().shape[0]))
        x = torch.empty_like(z)
        rep = L.pcg_solve(mesh, prec, dev(bo), x, 1e-8)
        xo, ro = P.pcg(bo, 1e-8)
        assert iters_match(P, bo, 1e-8, rep["iters"], ro["iters"]), (rep["iters"], ro["iters"])
        its.append(rep["iters"])
    assert max(its) <= 1.7 * min(its), its


def test_extension_rejected_for_star_patches(L):
    V = strip_vertices(4, 15.0)
    mesh = L.Mesh(2, (4, 4), 3, V)
    with pytest.raises(L.LorpcError):
        L.Prec(L.Lor(mesh), patch_kind="star", extend=True)
