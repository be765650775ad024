"""Pins of the oracle's non-affine (trilinear) geometry and of its coarse solver R_0.

VERDICT r01 "What's weak 1": every 3D operator / LOR pin was Cartesian (diagonal J,
vanishing off-diagonal cofactors) or self-consistency, and R_0 (reading c11) was
pinned by symmetry / SPD only.  The pins here use perturbed trilinear meshes of the
C5 recipe and quantities fixed by the mathematics, computed from data the oracle
does not produce (node coordinates from the vertex array and numpy GLL nodes):

* linear patch test (P:82-84 elements are images of the unit cube; eq:fem P:86-89):
  the coordinate functions x_k are reproduced exactly by the Q_p (K_p) and the
  subcell-Q1 (K_h) spaces on trilinear elements, so with the
  unconstrained stiffness K, x_k^T K x_l = int grad x_k . grad x_l = delta_kl |Omega|
  and (K x_k)_i = int d phi_i / d x_k = 0 for every interior node i.  Both are exact
  under the Gauss rules used (cofactors of a trilinear J are polynomials of degree
  <= 2 per variable).  A wrong sign / index in any 3D cofactor of det_inv, or a
  transposed J, breaks them.
* E^T A_IP E = K_FF on a perturbed 3D mesh (jumps of continuous functions vanish;
  eq:ip P:113-136) - the non-affine version of test_oracle_pins.py's Cartesian check.
* manufactured convergence of order p+1 on a perturbed 3D mesh (C3 solution on the C5
  perturbation recipe).
* R_0 is a uniform preconditioner for A_0 ("any scalable solver"; reading
  c11): kappa(R_0 A_0) from dense eigenvalues stays bounded as n doubles, in 2D and 3D.
"""
import dataclasses
import math

import numpy as np
import pytest
import scipy.linalg as sl

import oracle as O
from tests import indep
from workloads import CONFIGS, exact_solution, rhs_function, small_config, vertices

pytestmark = pytest.mark.filterwarnings("ignore")


def _perturbed(name, n, p, a):
    """The named recipe on n elements, degree p, interior vertices moved by U(-a h, a h)."""
    cfg = small_config(name, n, p=p)
    return dataclasses.replace(cfg, perturb=a, mesh_seed=CONFIGS["C5"].mesh_seed)


def _node_coords(cfg):
    """GLL node coordinates from the vertex array by the multilinear element map
    (numpy GLL nodes; no oracle call).  Global node grid x-fastest."""
    d, p, n = cfg.dim, cfg.p, cfg.n
    V = vertices(cfg).reshape([nk + 1 for nk in reversed(n)] + [d])   # [z][y][x][d] or [y][x][d]
    xi = indep.gll_nodes(p)
    N = [nk * p + 1 for nk in n]
    X = np.zeros((int(np.prod(N)), d))
    for g in range(X.shape[0]):
        c = [(g // int(np.prod(N[:k]))) % N[k] for k in range(d)]
        e = [min(c[k] // p, n[k] - 1) for k in range(d)]
        t = [xi[c[k] - e[k] * p] for k in range(d)]
        x = np.zeros(d)
        for corner in range(1 << d):
            b = [(corner >> k) & 1 for k in range(d)]
            w = np.prod([t[k] if b[k] else 1.0 - t[k] for k in range(d)])
            idx = tuple(e[k] + b[k] for k in reversed(range(d)))
            x += w * V[idx]
        X[g] = x
    return X, N


def _assembled_kp(P, cfg):
    """Unconstrained K_p = sum_e of the oracle's element matrices (local x-fastest)."""
    d, p, n = cfg.dim, cfg.p, cfg.n
    N = [nk * p + 1 for nk in n]
    nd = int(np.prod(N))
    K = np.zeros((nd, nd))
    nl = (p + 1) ** d
    for e in range(cfg.n_el):
        ec = [(e // int(np.prod(n[:k]))) % n[k] for k in range(d)]
        gid = np.zeros(nl, dtype=int)
        for a in range(nl):
            ac = [(a // (p + 1) ** k) % (p + 1) for k in range(d)]
            gid[a] = sum((ec[k] * p + ac[k]) * int(np.prod(N[:k])) for k in range(d))
        K[np.ix_(gid, gid)] += P.elem_matrix(e)
    return K


def _interior(N):
    return ~indep.boundary_mask(N)


def _linear_patch_checks(K, X, N):
    d = X.shape[1]
    scale = np.abs(K).max()
    G = X.T @ K @ X                       # x_k^T K x_l
    assert np.abs(G - np.eye(d)).max() < 1e-12, G          # |Omega| = 1 (boundary vertices fixed)
    inner = _interior(N)
    R = K @ X                             # (K x_k)_i
    assert np.abs(R[inner]).max() < 1e-12 * scale, np.abs(R[inner]).max()


@pytest.mark.parametrize("n,p", [((2, 2, 2), 2), ((3, 2, 2), 3), ((2, 2, 3), 2)])
def test_linear_patch_kp_trilinear_3d(n, p):
    cfg = _perturbed("C5", n, p, 0.25)
    P = O.Problem.from_config(cfg)
    X, N = _node_coords(cfg)
    # the oracle's own node map must agree with the independent one
    assert np.abs(P.node_coords() - X).max() < 1e-14
    _linear_patch_checks(_assembled_kp(P, cfg), X, N)


@pytest.mark.parametrize("n,p", [((2, 2, 2), 2), ((3, 2, 2), 3)])
def test_linear_patch_kh_trilinear_3d(n, p):
    cfg = _perturbed("C5", n, p, 0.25)
    P = O.Problem.from_config(cfg)
    P.lor_assemble()
    X, N = _node_coords(cfg)
    Kh = P.level_matrix(0).toarray()      # unconstrained subcell-Q1 stiffness on the GLL grid
    _linear_patch_checks(Kh, X, N)


def test_linear_patch_kp_bilinear_2d():
    cfg = _perturbed("C2", (3, 3), 4, 0.25)
    P = O.Problem.from_config(cfg)
    X, N = _node_coords(cfg)
    _linear_patch_checks(_assembled_kp(P, cfg), X, N)


def test_sipg_consistency_with_cg_perturbed_3d():
    """E^T A_IP E = K_FF on a trilinear (non-affine) mesh, penalty c = 10."""
    n, p = (2, 2, 2), 2
    base = _perturbed("C5", n, p, 0.2)
    V = vertices(base)
    c = 10.0
    A = O.Problem(3, n, p, V, disc="sipg", eta=(p + 1) ** 2 * c).assemble_dense()
    Pc = O.Problem(3, n, p, V)
    K = Pc.assemble_dense()
    X, N = _node_coords(base)
    free = _interior(N)
    nl = (p + 1) ** 3
    E = np.zeros((base.n_el * nl, Pc.ndof))
    for e in range(base.n_el):
        ex, ey, ez = e % n[0], (e // n[0]) % n[1], e // (n[0] * n[1])
        for a in range(nl):
            ax, ay, az = a % (p + 1), (a // (p + 1)) % (p + 1), a // (p + 1) ** 2
            g = (ex * p + ax) + N[0] * ((ey * p + ay) + N[1] * (ez * p + az))
            E[e * nl + a, g] = 1
    Ef = E[:, free]
    tol = max(1e-14, 1e-15 * c * (p + 1) ** 2) * 10
    assert np.abs(Ef.T @ A @ Ef - K[np.ix_(free, free)]).max() < tol * np.abs(K).max()
    assert np.abs(A - A.T).max() < 1e-12 * np.abs(A).max()


def test_manufactured_order_perturbed_3d():
    """u = sin sin sin on the C5 perturbation recipe: L2 error of order >= p + 0.8."""
    p, errs = 2, []
    for nn in (4, 8):
        cfg = _perturbed("C3", (nn,) * 3, p, 0.1)
        P = O.Problem.from_config(cfg)
        Xq = P.quad_points()
        b = P.rhs(rhs_function(cfg, Xq))
        P.schwarz_setup("vertex", "mdf", "gmg")
        u, _ = P.pcg(b, 1e-13)          # PCG is pinned against dense solves elsewhere
        errs.append(P.l2_error(u, exact_solution(cfg, Xq)))
    rate = math.log2(errs[0] / errs[1])
    assert rate >= p + 0.8, (errs, rate)


# ---------------------------------------------------------------- R_0 (reading c11)
def _vertex_prolongation(cfg, X_gll_free):
    """P_0: vertex grid -> GLL grid, multilinear hat weights in the GLL reference
    coordinate of each element, built from numpy GLL nodes."""
    d, p, n = cfg.dim, cfg.p, cfg.n
    xi = indep.gll_nodes(p)
    N = [nk * p + 1 for nk in n]
    nv = [nk + 1 for nk in n]
    P0 = np.zeros((int(np.prod(N)), int(np.prod(nv))))
    for g in range(P0.shape[0]):
        c = [(g // int(np.prod(N[:k]))) % N[k] for k in range(d)]
        e = [min(c[k] // p, n[k] - 1) for k in range(d)]
        t = [xi[c[k] - e[k] * p] for k in range(d)]
        for corner in range(1 << d):
            b = [(corner >> k) & 1 for k in range(d)]
            w = np.prod([t[k] if b[k] else 1.0 - t[k] for k in range(d)])
            v = sum((e[k] + b[k]) * int(np.prod(nv[:k])) for k in range(d))
            P0[g, v] += w
    return P0, N, nv


def _kappa_R0A0(cfg):
    P = O.Problem.from_config(cfg)
    P.lor_assemble()
    P.schwarz_setup("vertex", "mdf", "gmg")
    P0, N, nv = _vertex_prolongation(cfg, None)
    ff = _interior(N)
    cf = _interior(nv)
    Pf = P0[np.ix_(ff, cf)]
    Kh = P.level_matrix(0).toarray()[np.ix_(ff, ff)]
    A0 = Pf.T @ Kh @ Pf
    # B_c = P_0 R_0 P_0^T on the free fine nodes, column by column (which = 2: coarse term only)
    nd = P.ndof
    fidx = np.nonzero(ff)[0]
    Bc = np.zeros((fidx.size, fidx.size))
    for j, g in enumerate(fidx):
        e = np.zeros(nd)
        e[g] = 1.0
        Bc[:, j] = P.precond(e, which=2)[fidx]
    Pp = np.linalg.pinv(Pf)
    R0 = Pp @ Bc @ Pp.T
    assert np.abs(R0 - R0.T).max() < 1e-10 * np.abs(R0).max()
    ev = sl.eigh(A0, np.linalg.inv(R0), eigvals_only=True)   # spectrum of R_0 A_0
    assert ev[0] > 0
    return ev[-1] / ev[0], ev


def test_coarse_gmg_uniform_2d():
    kap = [_kappa_R0A0(small_config("C2", (nn, nn), p=2))[0] for nn in (4, 8, 16)]
    assert max(kap) < 4.0, kap
    assert kap[2] / kap[1] < 1.25, kap


def test_coarse_gmg_uniform_3d():
    kap = [_kappa_R0A0(_perturbed("C5", (nn,) * 3, 1, 0.1))[0] for nn in (4, 8)]
    assert max(kap) < 5.0, kap
    assert kap[1] / kap[0] < 1.5, kap


def test_coarse_gmg_exact_on_single_coarse_level():
    """n = 2: the vertex grid has one interior vertex, coarsening stops and R_0 is the
    exact inverse (dense Cholesky): kappa(R_0 A_0) = 1."""
    kap, ev = _kappa_R0A0(small_config("C2", (2, 2), p=3))
    assert abs(kap - 1.0) < 1e-10, ev
