"""Row f4 (sec:aniso; rem:anisotropy P:499-502): anisotropic strip
meshes and vertex patches extended for isotropic overlap (reading r6).  CPU only."""
import numpy as np
import pytest

import oracle as O
from workloads import small_config, strip_vertices, vertices


def element_aspects(V, n):
    Vv = V.reshape(n + 1, n + 1, 2)
    w = np.diff(Vv[:, :, 0], axis=1)[:-1, :]
    h = np.diff(Vv[:, :, 1], axis=0)[:, :-1]
    return np.maximum(w / h, h / w)


@pytest.mark.parametrize("aspect", [1.0, 1.5, 15.0, 1500.0])
def test_strip_mesh_aspect(aspect):
    """SPEC anisotropic_strip_mesh: aspect 1 -> uniform grid; otherwise the strip's
    elements have the requested aspect ratio (Fig. fig:aniso-mesh: 15), the rest
    stay near 1, element count fixed, all Jacobians positive."""
    n = 8
    V = strip_vertices(n, aspect)
    a = element_aspects(V, n)
    assert a.shape == (n, n)
    assert abs(a.max() - aspect) <= 1e-9 * aspect
    assert np.all(a[np.arange(n) != n // 2] < 1.2)
    if aspect == 1.0:
        assert np.allclose(V, vertices(small_config("C1", (n, n))), atol=1e-15)
    P = O.Problem(2, (n, n), 3, V)      # det J > 0 checked at every quadrature point
    P.elem_matrix(0)


def test_extension_inactive_on_isotropic_and_perturbed_meshes():
    """The H/2 trigger never fires on the uniform or the C2-perturbed (+-0.15h) meshes:
    the extended preconditioner is the unextended one, bit for bit."""
    for cfg in (small_config("C1", (5, 4), p=3), small_config("C2", (6, 5), p=4)):
        zs = []
        for ext in (False, True):
            P = O.Problem(2, cfg.n, cfg.p, vertices(cfg))
            P.schwarz_setup("vertex", "mdf", "gmg", extend=ext)
            r = np.random.default_rng(2).standard_normal(P.ndof)
            zs.append(P.precond(r))
        assert np.array_equal(zs[0], zs[1])


def test_extension_grows_strip_patches_by_one_layer():
    """Aspect 15: vertex patches touching the strip from one side get one more element
    row beyond it (3 rows); every other patch keeps its 2 x 2 (clipped) elements."""
    n = 8
    P = O.Problem(2, (n, n), 3, strip_vertices(n, 15.0))
    P.schwarz_setup("vertex", "mdf", "gmg", extend=True)
    r = n // 2
    for j in range(P.npatches()):
        vx, vy = j % (n + 1), j // (n + 1)
        lo, hi = P.patch_range(j)
        base_lo, base_hi = max(vy - 1, 0), min(vy, n - 1)
        assert lo[0] == max(vx - 1, 0) and hi[0] == min(vx, n - 1)
        if vy == r:            # strip row above the vertex: grow upwards
            assert (lo[1], hi[1]) == (base_lo, base_hi + 1)
        elif vy == r + 1:      # strip row below the vertex: grow downwards
            assert (lo[1], hi[1]) == (base_lo - 1, base_hi)
        else:
            assert (lo[1], hi[1]) == (base_lo, base_hi)


def test_extended_patches_make_iterations_aspect_independent():
    """Fig. fig:aniso-iters: with isotropic-overlap patches B(V) the PCG counts stay
    nearly constant from aspect 1.5 to 1500, while plain vertex patches degrade."""
    its = {}
    for ext in (False, True):
        its[ext] = []
        for a in (1.5, 15.0, 150.0, 1500.0):
            P = O.Problem(2, (8, 8), 3, strip_vertices(8, a))
            P.schwarz_setup("vertex", "mdf", "gmg", extend=ext)
            b = P.rhs(np.ones(P.quad_points().shape[0]))
            its[ext].append(P.pcg(b, 1e-8)[1]["iters"])
    assert max(its[True]) <= 1.7 * min(its[True]), its
    assert its[False][-1] >= 3 * its[False][0], its
