"""Quick GPU timing probe: setup, operator apply, preconditioner apply, PCG per config."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1908_07071_b200 import lorpc as L  # noqa: E402
from workloads import get_config, random_free_rhs, rhs_function, vertices  # noqa: E402


def timeit(fn, reps=10):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name in sys.argv[1:]:
    cfg = get_config(name)
    t = time.time()
    V = vertices(cfg)
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, V)
    torch.cuda.synchronize()
    t_mesh = time.time() - t
    t = time.time()
    lor = L.Lor(mesh)
    t_lor = time.time() - t
    t = time.time()
    prec = L.Prec(lor, patch_kind=cfg.patch_kind)
    t_prec = time.time() - t
    n = mesh.n_dof
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ta = timeit(lambda: mesh.apply(x, y))
    tp = timeit(lambda: prec.apply(x, y), reps=5)
    if cfg.rhs == "randn":
        b = torch.from_numpy(random_free_rhs(cfg)).cuda()
    else:
        xq = torch.empty(mesh.n_quad * cfg.dim, dtype=torch.float64, device="cuda")
        mesh.quad_points(xq)
        fq = torch.from_numpy(rhs_function(cfg, xq.cpu().numpy().reshape(-1, cfg.dim))).cuda()
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        mesh.rhs_assemble(fq, None, b)
    xs = torch.empty_like(b)
    rep = L.pcg_solve(mesh, prec, b, xs, cfg.tol)
    rep = L.pcg_solve(mesh, prec, b, xs, cfg.tol)
    it = rep["iters"]
    print(f"{name}: ndof={n} setup mesh {t_mesh:.2f}s lor {t_lor:.2f}s prec {t_prec:.2f}s | apply {ta*1e3:.1f} us"
          f" ({16*n/ta/1e6:.0f} GB/s x+y) precond {tp*1e3:.1f} us | pcg iters {it} {rep['t_solve_ms']:.2f} ms"
          f" -> {n*it/rep['t_solve_ms']*1e3:.3e} DOF-it/s  ({rep['t_solve_ms']/it*1e3:.0f} us/it)", flush=True)
    del prec, lor, mesh
    torch.cuda.empty_cache()
