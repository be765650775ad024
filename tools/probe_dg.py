"""GPU timing probe for the C4 SIPG configuration (three penalties)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1908_07071_b200 import lorpc as L  # noqa: E402
from workloads import dirichlet_function, get_config, rhs_function, small_config, vertices  # noqa: E402

cfg = get_config("C4") if len(sys.argv) < 2 else small_config("C4", tuple(int(v) for v in sys.argv[1].split(",")))
V = vertices(cfg)
for c in cfg.penalty_c:
    eta = (cfg.p + 1) ** 2 * c
    t = time.time()
    mesh = L.Mesh(3, cfg.n, cfg.p, V, disc=1, eta=eta)
    lor = L.Lor(mesh)
    prec = L.Prec(lor)
    torch.cuda.synchronize()
    ts = time.time() - t
    xq = torch.empty(mesh.n_quad * 3, dtype=torch.float64, device="cuda")
    xb = torch.empty(mesh.n_bface_quad * 3, dtype=torch.float64, device="cuda")
    mesh.quad_points(xq, xb)
    fq = torch.from_numpy(rhs_function(cfg, xq.cpu().numpy().reshape(-1, 3))).cuda()
    gq = torch.from_numpy(dirichlet_function(cfg, xb.cpu().numpy().reshape(-1, 3))).cuda()
    b = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    mesh.rhs_assemble(fq, gq, b)
    x = torch.empty_like(b)
    y = torch.empty_like(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mesh.apply(b, y)
    e0.record(); [mesh.apply(b, y) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    ta = e0.elapsed_time(e1) / 10
    prec.apply(b, y)
    e0.record(); [prec.apply(b, y) for _ in range(3)]; e1.record(); torch.cuda.synchronize()
    tp = e0.elapsed_time(e1) / 3
    rep = L.pcg_solve(mesh, prec, b, x, cfg.tol, cfg.maxit)
    print(f"C4 c={c}: ndof={mesh.n_dof} setup {ts:.2f}s apply {ta*1e3:.0f} us precond {tp*1e3:.0f} us "
          f"iters {rep['iters']} solve {rep['t_solve_ms']:.1f} ms -> {mesh.n_dof*rep['iters']/rep['t_solve_ms']*1e3:.3e} DOF-it/s",
          flush=True)
    del prec, lor, mesh
