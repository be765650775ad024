"""Multi-rank slab path on one GPU: all ranks emulated in one
process (lorpc_dist_create with nccl_id = NULL: the exchanges are device copies,
no kernels wait on each other).  The distributed operator, preconditioner and PCG
must reproduce the single-rank library path (same arithmetic up to summation
order: 1e-12) and the CPU oracle (PCG iterations +-1, solution 1e-9)."""
import numpy as np
import pytest

import oracle as O
from workloads import parity_vector, random_free_rhs, small_config, vertices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


# C5 recipe (trilinear, perturbed, random RHS) on small meshes; ranks up to n_z
CASES = [((4, 3, 5), 3, 2), ((4, 3, 5), 3, 5), ((3, 4, 7), 3, 3), ((3, 3, 6), 4, 2), ((3, 3, 4), 2, 4),
         ((4, 3, 8), 3, 8)]  # eight ranks of one element layer each (the 8-GPU C5 shape in miniature)


def split(D, v):
    return [dev(v[o:o + c]) for (o, c, _) in D.owned]


def join(D, parts, n):
    out = np.full(n, np.nan)
    for (o, c, _), t in zip(D.owned, parts):
        out[o:o + c] = t.cpu().numpy()
    return out


@pytest.mark.parametrize("n,p,R", CASES)
def test_dist_matches_single(L, n, p, R):
    cfg = small_config("C5", n, p=p)
    V = vertices(cfg)
    mesh = L.Mesh(3, cfg.n, p, V)
    prec = L.Prec(L.Lor(mesh))
    D = L.Dist(cfg.n, p, V, R)
    N = mesh.n_dof
    # ownership is a partition of the global node vector
    offs = sorted((o, c) for (o, c, _) in D.owned)
    assert offs[0][0] == 0 and sum(c for _, c in offs) == N
    assert all(offs[i][0] + offs[i][1] == offs[i + 1][0] for i in range(len(offs) - 1))
    assert sum(J for (_, _, J) in D.owned) == prec.n_patches
    x = parity_vector(N)
    # operator
    y1 = torch.empty(N, dtype=torch.float64, device="cuda")
    mesh.apply(dev(x), y1)
    ys = [torch.empty_like(t) for t in split(D, x)]
    D.apply(split(D, x), ys)
    torch.cuda.synchronize()
    assert rel(join(D, ys, N), y1.cpu().numpy()) < 1e-12
    # preconditioner (r with Dirichlet entries zeroed)
    P = O.Problem.from_config(cfg)
    X = P.node_coords()
    r = x.copy()
    r[~np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)] = 0.0
    z1 = torch.empty(N, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z1)
    zs = [torch.empty_like(t) for t in split(D, r)]
    D.precond(split(D, r), zs)
    torch.cuda.synchronize()
    assert rel(join(D, zs, N), z1.cpu().numpy()) < 1e-12
    # PCG: distributed vs single rank vs oracle
    b = random_free_rhs(cfg)
    x1 = torch.empty(N, dtype=torch.float64, device="cuda")
    rep1 = L.pcg_solve(mesh, prec, dev(b), x1, cfg.tol)
    xs = [torch.empty_like(t) for t in split(D, b)]
    repd = D.pcg_solve(split(D, b), xs, cfg.tol)
    xd = join(D, xs, N)
    assert abs(repd["iters"] - rep1["iters"]) <= 1, (repd["iters"], rep1["iters"])
    assert rel(xd, x1.cpu().numpy()) < 1e-9
    P.schwarz_setup("vertex", "mdf", "gmg")
    xo, ro = P.pcg(b, cfg.tol)
    assert abs(repd["iters"] - ro["iters"]) <= 1, (repd["iters"], ro["iters"])
    assert rel(xd, xo) < 1e-9


@pytest.mark.parametrize("n,p,R", [((4, 3, 5), 3, 2), ((4, 3, 8), 3, 8), ((3, 3, 4), 2, 4)])
def test_dist_rcm_matches_single(L, n, p, R):
    """The slab path with a structure-only ordering (RCM: the ranks' patch subsets run the
    U-record kernels, bench default of C5): preconditioner equal to the single-rank path,
    PCG iterations +-1 vs the single rank and the oracle."""
    cfg = small_config("C5", n, p=p)
    V = vertices(cfg)
    mesh = L.Mesh(3, cfg.n, p, V)
    prec = L.Prec(L.Lor(mesh), ordering="rcm")
    D = L.Dist(cfg.n, p, V, R, ordering="rcm")
    N = mesh.n_dof
    P = O.Problem.from_config(cfg)
    X = P.node_coords()
    r = parity_vector(N)
    r[~np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)] = 0.0
    z1 = torch.empty(N, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z1)
    zs = [torch.empty_like(t) for t in split(D, r)]
    D.precond(split(D, r), zs)
    torch.cuda.synchronize()
    assert rel(join(D, zs, N), z1.cpu().numpy()) < 1e-12
    b = random_free_rhs(cfg)
    x1 = torch.empty(N, dtype=torch.float64, device="cuda")
    rep1 = L.pcg_solve(mesh, prec, dev(b), x1, cfg.tol)
    xs = [torch.empty_like(t) for t in split(D, b)]
    repd = D.pcg_solve(split(D, b), xs, cfg.tol)
    xd = join(D, xs, N)
    assert abs(repd["iters"] - rep1["iters"]) <= 1, (repd["iters"], rep1["iters"])
    assert rel(xd, x1.cpu().numpy()) < 1e-9
    P.schwarz_setup("vertex", "rcm", "gmg")
    xo, ro = P.pcg(b, cfg.tol)
    assert abs(repd["iters"] - ro["iters"]) <= 1, (repd["iters"], ro["iters"])
    assert rel(xd, xo) < 1e-9


def test_dist_rejects_bad_partition(L):
    cfg = small_config("C5", (3, 3, 2), p=3)
    with pytest.raises(L.LorpcError):
        L.Dist(cfg.n, 3, vertices(cfg), 3)  # n_z < nranks


def test_dist_nccl_single_rank(L):
    """The NCCL transport (communicator, allreduces) on a 1-rank communicator:
    the only NCCL configuration one GPU can run; equals the single-rank path."""
    cfg = small_config("C5", (3, 4, 4), p=3)
    V = vertices(cfg)
    mesh = L.Mesh(3, cfg.n, 3, V)
    prec = L.Prec(L.Lor(mesh))
    D = L.Dist(cfg.n, 3, V, 1, rank=0, nccl_id=L.dist_nccl_id())
    b = random_free_rhs(cfg)
    x1 = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    rep1 = L.pcg_solve(mesh, prec, dev(b), x1, cfg.tol)
    xd = torch.empty_like(x1)
    repd = D.pcg_solve([dev(b)], [xd], cfg.tol)
    assert repd["iters"] == rep1["iters"]
    assert rel(xd.cpu().numpy(), x1.cpu().numpy()) < 1e-12


def test_dist_eight_ranks_c5_recipe_32cubed(L):
    """R = 8 emulated ranks of four element layers each on the C5 recipe at 32^3 (the
    8-GPU slab shape at 1/64 of the volume): operator and preconditioner equal the
    single-rank path to 1e-12, PCG iterations +-1 and the solution 1e-9 (the single-rank
    path itself is checked against the oracle at this size in test_gpu_large.py)."""
    cfg = small_config("C5", (32, 32, 32), p=3)
    V = vertices(cfg)
    mesh = L.Mesh(3, cfg.n, 3, V)
    prec = L.Prec(L.Lor(mesh))
    D = L.Dist(cfg.n, 3, V, 8)
    N = mesh.n_dof
    x = parity_vector(N, seed=56)
    y1 = torch.empty(N, dtype=torch.float64, device="cuda")
    mesh.apply(dev(x), y1)
    ys = [torch.empty_like(t) for t in split(D, x)]
    D.apply(split(D, x), ys)
    torch.cuda.synchronize()
    assert rel(join(D, ys, N), y1.cpu().numpy()) < 1e-12
    g = np.arange(N)
    Nx = cfg.n[0] * 3 + 1
    ix, iy, iz = g % Nx, (g // Nx) % Nx, g // (Nx * Nx)
    r = x.copy()
    r[(ix == 0) | (ix == Nx - 1) | (iy == 0) | (iy == Nx - 1) | (iz == 0) | (iz == Nx - 1)] = 0.0
    z1 = torch.empty(N, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z1)
    zs = [torch.empty_like(t) for t in split(D, r)]
    D.precond(split(D, r), zs)
    torch.cuda.synchronize()
    assert rel(join(D, zs, N), z1.cpu().numpy()) < 1e-12
    b = random_free_rhs(cfg)
    x1 = torch.empty(N, dtype=torch.float64, device="cuda")
    rep1 = L.pcg_solve(mesh, prec, dev(b), x1, cfg.tol)
    xs = [torch.empty_like(t) for t in split(D, b)]
    repd = D.pcg_solve(split(D, b), xs, cfg.tol)
    assert abs(repd["iters"] - rep1["iters"]) <= 1, (repd["iters"], rep1["iters"])
    assert rel(join(D, xs, N), x1.cpu().numpy()) < 1e-9
