"""Peer-store halo (NEXT-f3) on ONE GPU: 2 and 3 rank processes share cuda:0 and exchange their
halo rows through CUDA IPC buffers that the neighbours' pack kernels write into
(slab.PeerTransport / evaluate_rank_peer; host messages over gloo). No kernel waits on another
process: the ordering is stream-ordered interprocess events handed over by host messages.
The owned results must equal the single-context evaluation (and so the oracle)."""
import os
import socket

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, width, q):
    import torch
    import torch.distributed as dist

    import paper_1404_2303_b200 as sph
    from paper_1404_2303_b200 import slab
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        p = workloads.c1()
        edges = [k / world for k in range(world + 1)]
        lo, hi = edges[rank], edges[rank + 1]
        own = np.nonzero((p.x[:, 0] >= lo) & (p.x[:, 0] < hi))[0]
        h0 = np.full(p.n, 0.0704508, dtype=np.float32)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        cfg = sph.default_config(p.box, rank=rank, nranks=world, slab_lo=lo, slab_hi=hi, halo_width=width)
        ctx = sph.Context(cfg)
        tr = slab.PeerTransport(ctx, rank, world, cap_rows=p.n)
        out = []
        for _ in range(2):   # two evaluations: the buffers are reused after `consumed`
            r = slab.evaluate_rank_peer(ctx, t(p.x[own]), t(p.v[own]), t(p.m[own]), t(p.u[own]), t(h0[own]), lo,
                                        hi, width, tr)
            out.append({k: getattr(r, k).cpu().numpy() for k in ("h", "rho", "a", "dudt", "n_nbr", "n_nbr_force")})
            out[-1]["n_halo"] = r.n_halo
        torch.cuda.synchronize()
        q.put((rank, own, out))
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,width", [(2, 0.12), (3, 0.12), (3, 0.03)])
def test_peer_store_halo_matches_single_context(world, width):
    import torch.multiprocessing as mp

    from tests import parity
    p = workloads.c1()
    ref = parity.run_gpu(p)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, width, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    seen = np.zeros(p.n, int)
    scale = np.abs(ref["a"]).max()
    for rank in range(world):
        _, own, outs = res[rank]
        seen[own] += 1
        for o in outs:
            assert o["n_halo"] > 0
            assert np.allclose(o["h"], ref["h"][own], rtol=2e-6)
            assert np.allclose(o["rho"], ref["rho"][own], rtol=1e-5)
            assert np.array_equal(o["n_nbr"], ref["n_nbr"][own])
            assert np.array_equal(o["n_nbr_force"], ref["n_nbr_force"][own])
            assert np.abs(o["a"] - ref["a"][own]).max() <= 1e-4 * scale
        # the second evaluation reproduces the first bit for bit
        for k in ("h", "rho", "a", "dudt"):
            assert np.array_equal(outs[0][k], outs[1][k]), k
    assert np.all(seen == 1)
