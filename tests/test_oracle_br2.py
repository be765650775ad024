"""Pins of the oracle's BR2 DG operator (eq:br2 P:152-158, lifting eq:lift
P:662-665, reading c17) against an independent 1D construction (Kronecker
structure on Cartesian meshes, P:206-224 applied to the DG forms), and the
properties the paper states: symmetry, positive definiteness, BR2/IP norm
equivalence (Prop. after Lemma), penalty robustness of B_DG
(Cor. P:726-733)."""
import math

import numpy as np
import pytest
import scipy.linalg as sl

import oracle as O
from tests import indep
from tests.test_oracle_pins import _dg_perm
from workloads import dirichlet_function, exact_solution, rhs_function, small_config, vertices


def _br2(n, p, eta):
    cfg = small_config("C4", n, p=p)
    return cfg, O.Problem(3, cfg.n, cfg.p, vertices(cfg), disc="br2", eta=eta)


@pytest.mark.parametrize("eta", [1.0, 10.0])
def test_br2_equals_kronecker_of_1d_br2(eta):
    n, p = (2, 3, 2), 2
    cfg, P = _br2(n, p, eta)
    A = P.assemble_dense()
    mats = [indep.br2_1d(p, nk, eta) for nk in n]
    Ak = indep.kron_sum([m[0] for m in mats], [m[1] for m in mats])
    perm = _dg_perm(n, p)
    Ak = Ak[np.ix_(perm, perm)]
    assert np.abs(A - Ak).max() <= 1e-12 * np.abs(Ak).max()


def test_br2_symmetric_spd_penalty_monotone_and_diag():
    n, p = (2, 2, 2), 2
    cfg, P = _br2(n, p, 1.0)
    A = P.assemble_dense()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh(0.5 * (A + A.T))[0] > 0
    _, P2 = _br2(n, p, 2.0)
    Dd = P2.assemble_dense() - A
    assert np.linalg.eigvalsh(0.5 * (Dd + Dd.T))[0] > -1e-12 * np.abs(Dd).max()
    P.schwarz_setup("vertex", "mdf", "gmg")
    assert np.allclose(P.dg_diag(), np.diag(A), rtol=1e-12)


def test_br2_ip_norm_equivalence():
    """Prop.: ||.||_IP and ||.||_BR2 are equivalent; the generalized
    eigenvalues of (A_BR2, A_IP) at comparable penalties lie in a bounded interval
    that does not degenerate with p."""
    ratios = []
    for p in (1, 2, 3):
        cfg, Pb = _br2((2, 2, 2), p, 1.0)
        Pi = O.Problem(3, cfg.n, p, vertices(cfg), disc="sipg", eta=(p + 1) ** 2)
        Ab, Ai = Pb.assemble_dense(), Pi.assemble_dense()
        w = sl.eigh(0.5 * (Ab + Ab.T), 0.5 * (Ai + Ai.T), eigvals_only=True)
        assert w[0] > 0
        ratios.append(w[-1] / w[0])
    assert max(ratios) < 50 and ratios[-1] < 2 * ratios[0]


def test_br2_manufactured_order():
    errs = []
    p = 2
    for nn in (3, 6):
        cfg, P = _br2((nn,) * 3, p, 3.0)
        Xq = P.quad_points()
        b = P.rhs(rhs_function(cfg, Xq))
        P.rhs_bc(dirichlet_function(cfg, P.bface_points()), b)
        P.schwarz_setup("vertex", "mdf", "gmg")
        u, _ = P.pcg(b, 1e-12)
        errs.append(P.l2_error(u, exact_solution(cfg, Xq)))
    assert math.log2(errs[0] / errs[1]) >= p + 0.8


def test_br2_preconditioner_penalty_robust():
    """Cor.: kappa(B_DG A_BR2) bounded independently of eta."""
    ks = []
    for eta in (1.0, 10.0, 100.0, 1e3, 1e4):
        cfg, P = _br2((2, 2, 2), 2, eta)
        b = P.rhs(rhs_function(cfg, P.quad_points()))
        P.schwarz_setup("vertex", "mdf", "gmg")
        _, rep = P.pcg(b, 1e-10)
        ks.append(O.lanczos_kappa(rep["alpha"], rep["beta"]))
    assert max(ks) / min(ks) <= 2.0, ks
