"""Dev probe: preconditioner applies on the C5 recipe at a given size (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_07071_b200 import lorpc as L
from workloads import get_config, small_config, vertices
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = small_config("C5", (n, n, n)) if n != 128 else get_config("C5")
mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
prec = L.Prec(L.Lor(mesh), patch_kind=cfg.patch_kind)
r = torch.randn(mesh.n_dof, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
prec.apply(r, z)
prec.profile(True)
for _ in range(reps):
    prec.apply(r, z)
ms, k = prec.profile_read()
print(f"C5@{n}^3 patch V-cycle {ms / k:.3f} ms/apply", flush=True)
