import sys; sys.path.insert(0, '.')
import numpy as np, torch
import oracle as O
from paper_1908_07071_b200 import lorpc as L
from workloads import small_config, vertices, rhs_function
cfg = small_config("C4", (3, 3, 2), p=2); eta = 9 * 10.0
V = vertices(cfg)
mesh = L.Mesh(3, cfg.n, cfg.p, V, disc=1, eta=eta); lor = L.Lor(mesh); prec = L.Prec(lor)
P = O.Problem(3, cfg.n, cfg.p, V, disc="sipg", eta=eta); P.schwarz_setup("vertex", "mdf", "gmg")
bo = P.rhs(rhs_function(cfg, P.quad_points()))
x = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
rep = L.pcg_solve(mesh, prec, torch.from_numpy(bo).cuda(), x, 1e-10)
xo, ro = P.pcg(bo, 1e-10)
print(rep["iters"], ro["iters"])
n = min(len(rep["res"]), len(ro["res"]))
for k in range(0, n, max(1, n // 12)): print(k, rep["res"][k], ro["res"][k], abs(rep["res"][k]/ro["res"][k]-1))
print(rep["res"][-3:], ro["res"][-3:])
