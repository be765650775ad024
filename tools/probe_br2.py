"""BR2 penalty sweep on the C4 mesh (3D analog of Table tab:dg-penalty)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1908_07071_b200 import lorpc as L  # noqa: E402
from workloads import get_config, rhs_function, vertices  # noqa: E402

cfg = get_config("C4")
V = vertices(cfg)
for disc, name in [(2, "BR2"), (1, "IP")]:
    for eta in [1.0, 10.0, 100.0, 1e3, 1e4]:
        e = eta if disc == 2 else (cfg.p + 1) ** 2 * eta
        try:
            mesh = L.Mesh(3, cfg.n, cfg.p, V, disc=disc, eta=e)
        except L.LorpcError as ex:
            print(f"{name} eta={eta}: {ex}", flush=True)
            continue
        prec = L.Prec(L.Lor(mesh))
        xq = torch.empty(mesh.n_quad * 3, dtype=torch.float64, device="cuda")
        mesh.quad_points(xq)
        fq = torch.from_numpy(rhs_function(cfg, xq.cpu().numpy().reshape(-1, 3))).cuda()
        b = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
        mesh.rhs_assemble(fq, None, b)
        x = torch.empty_like(b)
        rep = L.pcg_solve(mesh, prec, b, x, 1e-8, 4000, allow_not_converged=True)
        print(f"{name} {'eta' if disc == 2 else 'c'}={eta}: iters {rep['iters']} (tol 1e-8, homogeneous data) "
              f"{rep['t_solve_ms']:.0f} ms", flush=True)
        del prec, mesh
