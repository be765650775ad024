"""Time the operator apply of one config with CUDA events (mesh only, no preconditioner)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1908_07071_b200 import lorpc as L  # noqa: E402
from workloads import get_config, vertices  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C5")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, vertices(cfg))
x = torch.rand(mesh.n_dof, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(5):
    mesh.apply(x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    mesh.apply(x, y)
e1.record()
torch.cuda.synchronize()
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'C5'} operator apply: {e0.elapsed_time(e1) / reps:.4f} ms")
