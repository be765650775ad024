"""The five BASELINE.json configurations (C1..C5) as plain data.

Citations: BASELINE.json "configs"; readings c9
(C1 element-star patches), c13 (SIPG penalty eta = (p+1)^2 * c), c18/c19 (seeds).
"""
from dataclasses import dataclass, field, replace
from typing import Tuple


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    n: Tuple[int, ...]          # elements per axis
    p: int                      # polynomial degree
    perturb: float = 0.0        # interior vertices moved by U(-a h, a h) per coordinate
    mesh_seed: int = 0
    rhs: str = "sin"            # "sin", "sincos" (C2), "expsin" (C4, weak BC), "randn" (C5)
    rhs_seed: int = 0
    disc: str = "cg"            # "cg" or "sipg"
    penalty_c: Tuple[float, ...] = ()   # SIPG: eta = (p+1)^2 * c
    patch_kind: str = "vertex"  # "vertex" (eq:patch) or "star" (reading c9)
    tol: float = 1e-10
    maxit: int = 2000

    @property
    def n_el(self) -> int:
        r = 1
        for v in self.n:
            r *= v
        return r

    @property
    def n_dof(self) -> int:
        """All nodes (metric convention, reading c20); DG: n_el (p+1)^d."""
        if self.disc == "cg":
            r = 1
            for v in self.n:
                r *= v * self.p + 1
            return r
        return self.n_el * (self.p + 1) ** self.dim


CONFIGS = {
    "C1": Config("C1", 2, (4, 4), 3, rhs="sin", patch_kind="star", tol=1e-10),
    "C2": Config("C2", 2, (64, 64), 7, perturb=0.15, mesh_seed=1908, rhs="sincos", tol=1e-10),
    "C3": Config("C3", 3, (32, 32, 32), 4, rhs="sin", tol=1e-10),
    "C4": Config("C4", 3, (32, 32, 32), 5, rhs="expsin", disc="sipg",
                 penalty_c=(1.0, 10.0, 1000.0), tol=1e-10),
    "C5": Config("C5", 3, (128, 128, 128), 3, perturb=0.1, mesh_seed=1909, rhs="randn",
                 rhs_seed=7071, tol=1e-8),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]


def shrink(cfg: Config, n: Tuple[int, ...], p: int = None) -> Config:
    """Same recipe on a smaller mesh (parity sizes the oracle finishes in seconds)."""
    return replace(cfg, name=f"{cfg.name}@{'x'.join(map(str, n))}", n=tuple(n),
                   p=cfg.p if p is None else p)
