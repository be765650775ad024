"""Profiling driver: set up one config and run operator + preconditioner applies."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1908_07071_b200 import lorpc as L  # noqa: E402
from workloads import get_config, small_config, vertices  # noqa: E402

# "C5m": the C5 recipe on 64^3 elements (faster ncu replays)
cfg = small_config("C5", (64, 64, 64)) if sys.argv[1] == "C5m" else get_config(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
lor = L.Lor(mesh)
prec = L.Prec(lor, patch_kind=cfg.patch_kind, ordering=sys.argv[3] if len(sys.argv) > 3 else "mdf")
x = torch.rand(mesh.n_dof, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(reps):
    mesh.apply(x, y)
    prec.apply(x, y)
torch.cuda.synchronize()
print("ok")
