"""Small end-to-end run of every hot-path kernel family (a quick crash / NaN check;
compute-sanitizer is closed on this pool):
CG operator + thread-mode V-cycle (C5 recipe, u8 and u16 records), group-mode
V-cycle (C2 recipe), PCG, and the slab decomposition emulated over 3 ranks."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1908_07071_b200 import lorpc as L  # noqa: E402
from workloads import random_free_rhs, small_config, vertices  # noqa: E402

for name, n, p in [("C5", (5, 4, 6), 3), ("C3", (3, 3, 4), 4), ("C2", (6, 5), 7)]:
    cfg = small_config(name, n, p=p)
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
    prec = L.Prec(L.Lor(mesh), patch_kind=cfg.patch_kind)
    x = torch.rand(mesh.n_dof, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    mesh.apply(x, y)
    prec.apply(x, y)
    b = torch.from_numpy(random_free_rhs(cfg)).cuda()  # b_D = 0 (the PCG convention)
    rep = L.pcg_solve(mesh, prec, b, y, 1e-8)
    assert rep["converged"] and torch.isfinite(y).all(), (name, rep["iters"])
    print(name, "iters", rep["iters"])
cfg = small_config("C5", (4, 3, 6), p=3)
V = vertices(cfg)
D = L.Dist(cfg.n, 3, V, 3)
bb = random_free_rhs(cfg)
bs = [torch.from_numpy(np.ascontiguousarray(bb[o:o + c])).cuda() for (o, c, _) in D.owned]
xs = [torch.empty_like(t) for t in bs]
rep = D.pcg_solve(bs, xs, 1e-8)
assert rep["converged"]
torch.cuda.synchronize()
print("ok")
