"""Helpers shared by the GPU parity tests (expected values only from oracle/)."""
import numpy as np


def oracle_iter_band(P, b, tol, k=6):
    """Range of the oracle's PCG iteration counts over b and k copies of b perturbed
    by 1e-15 relative noise: the oracle's own rounding floor for the iteration count
    (where the residual stagnates next to tol a rounding-level change of the input
    already moves the crossing; reading r2)."""
    rng = np.random.default_rng(1234)
    its = [P.pcg(b, tol)[1]["iters"]]
    for _ in range(k):
        its.append(P.pcg(b * (1 + 1e-15 * rng.standard_normal(b.shape)), tol)[1]["iters"])
    return min(its), max(its)


def iters_match(P, b, tol, gpu_iters, oracle_iters):
    """GPU PCG iterations within +-1 of the oracle's; only if not, within +-1 of the
    oracle's own rounding band (oracle_iter_band)."""
    if abs(gpu_iters - oracle_iters) <= 1:
        return True
    lo, hi = oracle_iter_band(P, b, tol)
    return lo - 1 <= gpu_iters <= hi + 1
