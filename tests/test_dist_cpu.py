"""The N > 1 path's host logic on CPU, world_size 2 and 3 over gloo: the slab
plans the C library computes (lorpc_dist_plan_get, the plan dist.cu executes)
partition the node and vertex planes, and the four exchange phases, run here as
gloo send / recv of numpy planes, deliver exactly the global values (copy phases)
and the neighbour sums (add phases) each rank's kernels read."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nz, p, plane, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1908_07071_b200 import lorpc as L
        P = L.dist_plan(nz, p, world, rank)
        G = nz * p + 1  # global node planes
        rng = np.random.default_rng(7)
        g = rng.standard_normal((G, plane))  # the global vector, identical on every rank
        nloc = (P["zb"] - P["za"]) * p + 1
        base = P["za"] * p  # global plane of local plane 0
        # ownership partition (gathered)
        own = torch.tensor([P["gown_plane0"], P["own_planes"], P["own_plane0"] + base, P["nvown"],
                            P["vown0"] + P["za"]], dtype=torch.int64)
        allown = [torch.zeros_like(own) for _ in range(world)]
        dist.all_gather(allown, own)
        planes = sorted((int(a[0]), int(a[1])) for a in allown)
        assert planes[0][0] == 0 and sum(c for _, c in planes) == G
        assert all(planes[i][0] + planes[i][1] == planes[i + 1][0] for i in range(world - 1))
        assert all(int(a[0]) == int(a[2]) for a in allown)
        vpl = sorted((int(a[4]), int(a[3])) for a in allown)
        assert vpl[0][0] == 0 and sum(c for _, c in vpl) == nz + 1
        assert P["z0"] * p == P["gown_plane0"] and P["za"] <= max(P["z0"] - 1, 0) and P["zb"] <= nz

        def run(k, loc):
            """phase k on the local array loc [nloc][plane] (gloo point-to-point)."""
            n = P["nplanes"][k]
            if n == 0:
                return
            reqs = []
            if P["to"][k] >= 0:
                s0 = P["send0"][k]
                reqs.append(dist.isend(torch.from_numpy(loc[s0:s0 + n].copy()), P["to"][k]))
            if P["from"][k] >= 0:
                buf = torch.zeros((n, plane), dtype=torch.float64)
                dist.recv(buf, P["from"][k])
                r0 = P["recv0"][k]
                if k in (1, 3):
                    loc[r0:r0 + n] += buf.numpy()
                else:
                    loc[r0:r0 + n] = buf.numpy()
            for rq in reqs:
                rq.wait()

        o0, no = P["own_plane0"], P["own_planes"]
        # E1 (operator input): owned planes + plane z1 p must hold the global values
        loc = np.full((nloc, plane), np.nan)
        loc[o0:o0 + no] = g[base + o0: base + o0 + no]
        run(0, loc)
        hi = (P["z1"] - P["za"]) * p
        assert np.array_equal(loc[o0:hi + 1], g[base + o0: base + hi + 1])
        # E3 (Schwarz input): planes (z0-1)p+1 .. z1 p - 1 must hold the global values
        loc = np.full((nloc, plane), np.nan)
        loc[o0:o0 + no] = g[base + o0: base + o0 + no]
        run(2, loc)
        lo = max((P["z0"] - 1 - P["za"]) * p + 1, 0)
        top = (P["z1"] - P["za"]) * p - 1
        assert np.array_equal(loc[lo:top + 1], g[base + lo: base + top + 1])
        # E2 / E4 (add): every rank contributes 1 to each local plane it touches;
        # after the exchange an owned plane holds its number of contributors
        loc = np.zeros((nloc, plane))
        e_lo, e_hi = (P["z0"] - P["za"]) * p, (P["z1"] - P["za"]) * p  # owned elements' node planes
        loc[e_lo:e_hi + 1] = 1.0
        run(1, loc)
        want = np.ones(no)
        gpl = np.arange(P["gown_plane0"], P["gown_plane0"] + no)
        interfaces = {int(a[0]) for a in allown if int(a[0]) > 0}
        want[np.isin(gpl, list(interfaces))] = 2.0
        assert np.array_equal(loc[o0:o0 + no, 0], want)
        loc = np.zeros((nloc, plane))
        lo_p = max((P["z0"] - 1 - P["za"]) * p + 1, 0)
        loc[lo_p:(P["z1"] - P["za"]) * p] = 1.0  # patch boxes of the owned vertex planes
        run(3, loc)
        # an owned plane g holds 1 from the rank's own patches (g <= z1 p - 1) plus 1 from
        # the next rank's patches (its boxes reach down to (z1 - 1) p + 1)
        gpl = np.arange(P["gown_plane0"], P["gown_plane0"] + no)
        want = (gpl <= P["z1"] * p - 1).astype(float)
        if P["from"][3] >= 0:
            want += (gpl >= (P["z1"] - 1) * p + 1)
        assert np.array_equal(loc[o0:o0 + no, 0], want)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world,nz,p", [(2, 5, 3), (3, 7, 4), (2, 2, 2)])
def test_slab_plan_exchanges_gloo(world, nz, p):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, p, 6, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    bad = [m for _, m in res if m != "ok"]
    assert not bad, bad[0]
