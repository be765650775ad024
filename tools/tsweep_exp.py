"""Time the preconditioner apply of one config under several LORPC_T* settings."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1908_07071_b200 import lorpc as L  # noqa: E402
from workloads import get_config, vertices  # noqa: E402

cfg = get_config(sys.argv[1])
mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
lor = L.Lor(mesh)
prec = L.Prec(lor, patch_kind=cfg.patch_kind)
x = torch.rand(mesh.n_dof, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for spec in sys.argv[2:]:
    for kv in spec.split(","):
        k, v = kv.split("=")
        os.environ[k] = v
    prec.apply(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        prec.apply(x, y)
    e1.record()
    torch.cuda.synchronize()
    print(f"{spec}: {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
