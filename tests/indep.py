"""Independent textbook constructions used to pin the oracle (tests only).

Nothing here is shared with oracle/ or the CUDA path: GLL / Gauss rules come
from numpy.polynomial.legendre, Lagrange polynomials from a Vandermonde solve,
and the 1D finite-element matrices from their definitions; d-dimensional
Cartesian operators from Kronecker products.
"""
import numpy as np
from numpy.polynomial import legendre as L


def gll_nodes(p):
    """GLL nodes on [0,1]: endpoints plus roots of P_p' (numpy root finder)."""
    c = np.zeros(p + 1)
    c[p] = 1.0
    r = L.legroots(L.legder(c)) if p > 1 else np.array([])
    t = np.concatenate([[-1.0], np.sort(r), [1.0]])
    return 0.5 * (t + 1.0)


def gauss(q):
    t, w = L.leggauss(q)
    return 0.5 * (t + 1.0), 0.5 * w


def lagrange_tables(nodes, pts):
    """Values and derivatives of the nodal Lagrange basis at pts (scipy barycentric)."""
    from scipy.interpolate import BarycentricInterpolator
    n = len(nodes)
    Bv = np.zeros((len(pts), n))
    Dv = np.zeros((len(pts), n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        f = BarycentricInterpolator(nodes, e)
        Bv[:, j] = f(pts)
        Dv[:, j] = f.derivative(pts, 1)
    return Bv, Dv


def fe_1d(p, n, length=1.0):
    """1D high-order stiffness / mass on n equal elements (Gauss q=p+1), global GLL grid."""
    xi = gll_nodes(p)
    xg, wg = gauss(p + 1)
    B, D = lagrange_tables(xi, xg)
    h = length / n
    Ke = D.T @ np.diag(wg) @ D / h
    Me = B.T @ np.diag(wg) @ B * h
    N = n * p + 1
    K = np.zeros((N, N))
    M = np.zeros((N, N))
    for e in range(n):
        s = slice(e * p, e * p + p + 1)
        K[s, s] += Ke
        M[s, s] += Me
    return K, M


def p1_1d(points):
    """Piecewise-linear stiffness / mass on a 1D grid of points (exact integrals)."""
    N = len(points)
    K = np.zeros((N, N))
    M = np.zeros((N, N))
    for i in range(N - 1):
        h = points[i + 1] - points[i]
        K[i:i + 2, i:i + 2] += np.array([[1, -1], [-1, 1]]) / h
        M[i:i + 2, i:i + 2] += np.array([[2, 1], [1, 2]]) * h / 6
    return K, M


def gll_grid_points(p, n, retained=None):
    xi = gll_nodes(p)
    if retained is not None:
        xi = xi[list(retained)]
    pts = [0.0]
    for e in range(n):
        pts.extend(list((e + xi[1:]) / n))
    return np.array(pts)


def kron_sum(Ks, Ms):
    """sum_j (x)_i G_i^j with G = K in slot j and M elsewhere; slot 0 = x (fastest)."""
    d = len(Ks)
    total = 0
    for j in range(d):
        mats = [Ks[i] if i == j else Ms[i] for i in range(d)]
        # x-fastest ordering: kron(z, kron(y, x))
        A = mats[0]
        for i in range(1, d):
            A = np.kron(mats[i], A)
        total = total + A
    return total


def boundary_mask(N_axes):
    grids = np.meshgrid(*[np.arange(v) for v in reversed(N_axes)], indexing="ij")
    coords = [g.ravel() for g in reversed(grids)]
    mask = np.zeros(coords[0].size, dtype=bool)
    for k, c in enumerate(coords):
        mask |= (c == 0) | (c == N_axes[k] - 1)
    return mask


def sipg_1d(p, n, sigma_c):
    """1D SIPG (Gauss q=p+1) on n equal elements of [0,1], sigma = sigma_c / h,
    Dirichlet imposed weakly at both ends; plus the DG mass.  Element-major."""
    xi = gll_nodes(p)
    xg, wg = gauss(p + 1)
    B, D = lagrange_tables(xi, xg)
    e0, de0 = lagrange_tables(xi, np.array([0.0, 1.0]))
    h = 1.0 / n
    sigma = sigma_c / h
    nl = p + 1
    A = np.zeros((n * nl, n * nl))
    M = np.zeros((n * nl, n * nl))
    for e in range(n):
        s = slice(e * nl, (e + 1) * nl)
        A[s, s] += D.T @ np.diag(wg) @ D / h
        M[s, s] += B.T @ np.diag(wg) @ B * h
    # trace values and d/dx at the left (0) and right (1) end of an element
    vL, vR = e0[0], e0[1]
    dL, dR = de0[0] / h, de0[1] / h
    for f in range(n + 1):
        # face at x = f h; K^- = element f-1 (right end), K^+ = element f (left end)
        # jump [v] = v^- - v^+ (normal +1 from K^-), avg {v'} = (v'^- + v'^+)/2
        jm = np.zeros(n * nl)
        av = np.zeros(n * nl)
        if f > 0 and f < n:
            jm[(f - 1) * nl:f * nl] += vR
            jm[f * nl:(f + 1) * nl] -= vL
            av[(f - 1) * nl:f * nl] += 0.5 * dR
            av[f * nl:(f + 1) * nl] += 0.5 * dL
        elif f == 0:      # boundary, outward normal -1: [v] = -v, {v'} = v'
            jm[0:nl] = -vL
            av[0:nl] = dL
        else:             # boundary at x = 1, outward normal +1
            jm[(n - 1) * nl:] = vR
            av[(n - 1) * nl:] = dR
        A += -np.outer(jm, av) - np.outer(av, jm) + sigma * np.outer(jm, jm)
    return A, M


def br2_1d(p, n, eta):
    """1D BR2 (Gauss q=p+1) on n equal elements of [0,1], weak Dirichlet at both ends.
    The lifting of a point jump into element K is r = -s_K M_K^{-1} (J n psi^K(x_e)),
    so eta (r_e[u], r_e[v]) = eta J(u) J(v) sum_K s_K^2 (M_K^{-1})_{end,end}
    (s = 1/2 interior, 1 boundary).  Built from the SIPG form with sigma replaced."""
    xi = gll_nodes(p)
    xg, wg = gauss(p + 1)
    B, D = lagrange_tables(xi, xg)
    e0, de0 = lagrange_tables(xi, np.array([0.0, 1.0]))
    h = 1.0 / n
    nl = p + 1
    Mref = B.T @ np.diag(wg) @ B
    Minv = np.linalg.inv(Mref * h)
    A = np.zeros((n * nl, n * nl))
    M = np.zeros((n * nl, n * nl))
    for e in range(n):
        s = slice(e * nl, (e + 1) * nl)
        A[s, s] += D.T @ np.diag(wg) @ D / h
        M[s, s] += Mref * h
    vL, vR = e0[0], e0[1]
    dL, dR = de0[0] / h, de0[1] / h
    for f in range(n + 1):
        jm = np.zeros(n * nl)
        av = np.zeros(n * nl)
        if 0 < f < n:
            jm[(f - 1) * nl:f * nl] += vR
            jm[f * nl:(f + 1) * nl] -= vL
            av[(f - 1) * nl:f * nl] += 0.5 * dR
            av[f * nl:(f + 1) * nl] += 0.5 * dL
            pen = eta * 0.25 * (Minv[p, p] + Minv[0, 0])
        elif f == 0:
            jm[0:nl] = -vL
            av[0:nl] = dL
            pen = eta * Minv[0, 0]
        else:
            jm[(n - 1) * nl:] = vR
            av[(n - 1) * nl:] = dR
            pen = eta * Minv[p, p]
        A += -np.outer(jm, av) - np.outer(av, jm) + pen * np.outer(jm, jm)
    return A, M


# ---------------------------------------------------------------- weighted 1D matrices (row f3 pins)
def fe_1d_weighted(p, n, bfun, length=1.0, extra=3):
    """1D high-order stiffness and mass with weight b(x), integrated with a Gauss rule
    of p+1+extra points per element (exact for polynomial b of degree <= 2 extra)."""
    xi = gll_nodes(p)
    tg, wg = gauss(p + 1 + extra)
    B, D = lagrange_tables(xi, tg)
    h = length / n
    N = n * p + 1
    K = np.zeros((N, N))
    M = np.zeros((N, N))
    for e in range(n):
        bw = wg * bfun(e * h + h * tg)
        s = slice(e * p, e * p + p + 1)
        K[s, s] += D.T @ np.diag(bw) @ D / h
        M[s, s] += B.T @ np.diag(bw) @ B * h
    return K, M


def p1_1d_weighted(points, bfun):
    """Piecewise-linear stiffness / mass with weight b(x) on a 1D grid (4-point Gauss
    per interval: exact for b of degree <= 5)."""
    tg, wg = gauss(4)
    N = len(points)
    K = np.zeros((N, N))
    M = np.zeros((N, N))
    for i in range(N - 1):
        a, h = points[i], points[i + 1] - points[i]
        x = a + h * tg
        bw = wg * bfun(x)
        phi = np.stack([1 - tg, tg])
        dphi = np.array([-1.0, 1.0]) / h
        K[i:i + 2, i:i + 2] += np.outer(dphi, dphi) * bw.sum() * h
        M[i:i + 2, i:i + 2] += (phi * bw) @ phi.T * h
    return K, M
