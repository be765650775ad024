"""Seeded input generators (vertex arrays, RHS functions, random vectors).

No method arithmetic lives here: only the problem data of SURVEY.md §8(d)
"Synthetic inputs" and readings c18/c19.  RNG: numpy Generator(PCG64(seed)).
"""
import math

import numpy as np

from .configs import Config, shrink


def vertices(cfg: Config) -> np.ndarray:
    """Vertex array [(n0+1)(n1+1)(n2+1), d], x-fastest, on [0,1]^d.

    Reading c18: interior vertices only are perturbed, one U(-a h, a h) draw per
    coordinate, vertices visited x-fastest, (dx, dy[, dz]) per vertex.
    """
    d = cfg.dim
    axes = [np.arange(n + 1, dtype=np.float64) / n for n in cfg.n]
    if d == 2:
        Y, X = np.meshgrid(axes[1], axes[0], indexing="ij")
        V = np.stack([X.ravel(), Y.ravel()], axis=1)
        idx = [np.arange(cfg.n[0] + 1)[None, :].repeat(cfg.n[1] + 1, 0).ravel(),
               np.arange(cfg.n[1] + 1)[:, None].repeat(cfg.n[0] + 1, 1).ravel()]
    else:
        Z, Y, X = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
        V = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
        i0 = np.arange(cfg.n[0] + 1)
        i1 = np.arange(cfg.n[1] + 1)
        i2 = np.arange(cfg.n[2] + 1)
        K, J, I = np.meshgrid(i2, i1, i0, indexing="ij")
        idx = [I.ravel(), J.ravel(), K.ravel()]
    V = np.ascontiguousarray(V)
    if cfg.perturb > 0.0:
        interior = np.ones(V.shape[0], dtype=bool)
        for k in range(d):
            interior &= (idx[k] > 0) & (idx[k] < cfg.n[k])
        rng = np.random.Generator(np.random.PCG64(cfg.mesh_seed))
        ids = np.nonzero(interior)[0]
        h = np.array([1.0 / n for n in cfg.n])
        delta = rng.uniform(-1.0, 1.0, size=(ids.size, d)) * (cfg.perturb * h)[None, :]
        V[ids] += delta
    return V


def exact_solution(cfg: Config, X: np.ndarray) -> np.ndarray:
    x = X[:, 0]
    y = X[:, 1]
    pi = math.pi
    if cfg.rhs == "sin":
        u = np.sin(pi * x) * np.sin(pi * y)
        if cfg.dim == 3:
            u = u * np.sin(pi * X[:, 2])
        return u
    if cfg.rhs == "sincos":
        return np.sin(pi * x) * np.sin(pi * y) * np.cos(pi * x * y)
    if cfg.rhs == "expsin":
        return np.exp(x) * np.sin(pi * y) * np.sin(pi * X[:, 2])
    raise ValueError(f"no exact solution for rhs={cfg.rhs}")


def rhs_function(cfg: Config, X: np.ndarray) -> np.ndarray:
    """f = -Laplace(u) for the manufactured solutions of BASELINE.json."""
    x = X[:, 0]
    y = X[:, 1]
    pi = math.pi
    if cfg.rhs == "sin":
        return cfg.dim * pi * pi * exact_solution(cfg, X)
    if cfg.rhs == "sincos":
        # f = pi^2[(2+x^2+y^2) sin(pi x)sin(pi y)cos(pi xy)
        #                 + 2 sin(pi xy)(y cos(pi x) sin(pi y) + x sin(pi x) cos(pi y))]
        return pi * pi * ((2 + x * x + y * y) * np.sin(pi * x) * np.sin(pi * y) * np.cos(pi * x * y)
                          + 2 * np.sin(pi * x * y) * (y * np.cos(pi * x) * np.sin(pi * y)
                                                      + x * np.sin(pi * x) * np.cos(pi * y)))
    if cfg.rhs == "expsin":
        return (2 * pi * pi - 1.0) * exact_solution(cfg, X)
    raise ValueError(f"no forcing for rhs={cfg.rhs}")


def dirichlet_function(cfg: Config, X: np.ndarray) -> np.ndarray:
    """g = u on the boundary (C4 weak Dirichlet data, reading c15)."""
    return exact_solution(cfg, X)


def random_free_rhs(cfg: Config) -> np.ndarray:
    """C5: b_i ~ N(0,1) on free nodes in lexicographic order, b_D = 0 (reading c19)."""
    N = [n * cfg.p + 1 for n in cfg.n]
    grids = np.meshgrid(*[np.arange(v) for v in reversed(N)], indexing="ij")
    coords = [g.ravel() for g in reversed(grids)]  # x-fastest
    free = np.ones(coords[0].size, dtype=bool)
    for k, c in enumerate(coords):
        free &= (c > 0) & (c < N[k] - 1)
    rng = np.random.Generator(np.random.PCG64(cfg.rhs_seed))
    b = np.zeros(coords[0].size)
    b[free] = rng.standard_normal(int(free.sum()))
    return b


def parity_vector(n: int, seed: int = 42) -> np.ndarray:
    """Per-apply parity input: x ~ U(-1,1) per entry."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=n)


def small_config(name: str, n, p=None) -> Config:
    from .configs import CONFIGS
    return shrink(CONFIGS[name], tuple(n), p)


# ------------------------------------------------------------------ variable coefficients (row f3)
COEFF_SEED = 9011


def coefficient_function(kind: str, X: np.ndarray) -> np.ndarray:
    """b(x, y) of -div(b grad u) (sec:variable-coeff).  The paper's
    domain is [-1,1]^2; ours is [0,1]^d, mapped by x' = 2x - 1 (reading r4).
      b1 = 1e4 (1 - x'^2)(1 - y'^2), b2 = 100 x'^2 + y'^2 + 1, b3 = (1 + x'^2 + y'^2)^4."""
    xp = 2.0 * X[:, 0] - 1.0
    yp = 2.0 * X[:, 1] - 1.0
    if kind == "b1":
        return 1e4 * (1.0 - xp * xp) * (1.0 - yp * yp)
    if kind == "b2":
        return 100.0 * xp * xp + yp * yp + 1.0
    if kind == "b3":
        return (1.0 + xp * xp + yp * yp) ** 4
    if kind == "one":
        return np.ones(X.shape[0])
    raise ValueError(kind)


def coefficient_b4(n_el: int, seed: int = COEFF_SEED) -> np.ndarray:
    """b4: piecewise constant, 10 or 1 per element, drawn at random;
    i.i.d. fair draws with PCG64(seed), elements in x-fastest order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.where(rng.random(n_el) < 0.5, 10.0, 1.0)


def coefficient_samples(kind: str, cfg: Config, Xq: np.ndarray, Xs: np.ndarray):
    """(b at the volume quadrature points, b at the LOR subcell Gauss points) for
    coefficient `kind`.  Xq is [n_el * q^d, d] element-major (the layout of
    quad_points), Xs is [n_sub * 2^d, d] with the global subcell index
    sx + (N0-1)(sy + (N1-1) sz) major (the layout of subcell_points).  b4 needs no
    coordinates: each point takes its element's value."""
    if kind != "b4":
        return coefficient_function(kind, Xq), coefficient_function(kind, Xs)
    be = coefficient_b4(cfg.n_el)
    nq = Xq.shape[0] // cfg.n_el
    bq = np.repeat(be, nq)
    d, p = cfg.dim, cfg.p
    Ns = [n * p for n in cfg.n]                       # subcells per axis
    ns = int(np.prod(Ns))
    s = np.arange(ns)
    sc = [s % Ns[0], (s // Ns[0]) % Ns[1]] + ([s // (Ns[0] * Ns[1])] if d == 3 else [])
    ec = [c // p for c in sc]
    e = ec[0] + cfg.n[0] * (ec[1] + (cfg.n[1] * ec[2] if d == 3 else 0))
    bs = np.repeat(be[e], 1 << d)
    return bq, bs


# ------------------------------------------------------------------ anisotropic strip meshes (row f4)
def strip_vertices(n: int, aspect: float, row: int = None) -> np.ndarray:
    """2D n x n Cartesian-topology mesh of [0,1]^2 whose element row `row` (default
    n // 2) is compressed to height 1/(n aspect), so its elements have aspect ratio
    `aspect`; the other rows share the remaining height equally (P:1107-1121,
    sec:aniso: "a strip of high-aspect-ratio elements"; SPEC's
    anisotropic_strip_mesh).  Vertices x-fastest, [(n+1)^2, 2]."""
    if aspect < 1.0:
        raise ValueError("aspect must be >= 1")
    r = n // 2 if row is None else row
    hs = 1.0 / (n * aspect)
    if n > 1:
        ho = (1.0 - hs) / (n - 1)
        heights = np.full(n, ho)
        heights[r] = hs
    else:
        heights = np.array([1.0])
    y = np.concatenate([[0.0], np.cumsum(heights)])
    y[-1] = 1.0
    x = np.arange(n + 1) / n
    X, Y = np.meshgrid(x, y, indexing="xy")
    return np.stack([X.ravel(), Y.ravel()], axis=1)
