"""Dev probe: W-mode (vcycle_w.cu) preconditioner vs the oracle on small C5-recipe
meshes, and the C5 full-size preconditioner apply time (W mode vs thread mode)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_1908_07071_b200 import lorpc as L
from workloads import get_config, parity_vector, small_config, vertices

def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()

def parity(cfg):
    V = vertices(cfg)
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, V)
    prec = L.Prec(L.Lor(mesh), patch_kind=cfg.patch_kind)
    P = O.Problem.from_config(cfg)
    P.schwarz_setup(cfg.patch_kind, "mdf", "gmg")
    r = parity_vector(P.ndof, seed=43)
    X = P.node_coords()
    free = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    r[~free] = 0.0
    z = torch.empty(mesh.n_dof, dtype=torch.float64, device="cuda")
    prec.apply(dev(r), z)
    zo = P.precond(r)
    zg = z.cpu().numpy()
    print(cfg.name, "rel", np.linalg.norm(zg - zo) / np.linalg.norm(zo), "maxabs",
          np.abs(zg - zo).max() / np.abs(zo).max(), flush=True)

def timing(wmode):
    os.environ["LORPC_WMODE"] = str(wmode)
    cfg = get_config(os.environ.get("WCFG", "C5"))
    V = vertices(cfg)
    t0 = time.time()
    mesh = L.Mesh(cfg.dim, cfg.n, cfg.p, V)
    prec = L.Prec(L.Lor(mesh), patch_kind=cfg.patch_kind)
    torch.cuda.synchronize()
    t1 = time.time()
    r = torch.randn(mesh.n_dof, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    for _ in range(3):
        prec.apply(r, z)
    prec.profile(True)
    for _ in range(10):
        prec.apply(r, z)
    ms, n = prec.profile_read()
    print(f"wmode={wmode} setup {t1-t0:.1f}s patch V-cycle {ms/n:.3f} ms/apply  |z|={z.norm().item():.6e}", flush=True)
    return z.cpu()

if __name__ == "__main__":
    for cfg in [small_config("C5", (4, 3, 5)), small_config("C3", (4, 3, 3), p=2), small_config("C5", (8, 8, 8)),
                small_config("C5", (2, 2, 2)), small_config("C5", (1, 3, 2))]:
        parity(cfg)
    if len(sys.argv) > 1:
        za = timing(1)
        zb = timing(0)
        print("W vs T rel diff", ((za - zb).norm() / zb.norm()).item())
