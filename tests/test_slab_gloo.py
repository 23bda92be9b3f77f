"""Multi-rank (N > 1) path on the CPU: world-size-2 gloo process group.

Checks the slab machinery that is not device arithmetic: count-quantile cuts, the
neighbour exchange over torch.distributed P2P (message matching when both neighbours are
the same rank, zero-length messages), and that owned + received-halo particles reproduce
the global result: each rank runs the fp64 oracle on its owned targets with its halo as
extra sources and the gathered per-rank results equal the oracle on the whole box.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_1404_2303_b200 import slab


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_cuts_quantiles():
    hist = np.array([10, 0, 0, 30, 40, 20])
    e = slab.slab_cuts(hist, 0.0, 6.0, 4)
    assert e[0] == 0.0 and e[-1] == 6.0 and np.all(np.diff(e) > 0)
    cum = np.concatenate([[0], np.cumsum(hist)])
    for k in range(1, 4):   # each cut splits the counts at k/4 (linear inside a bin)
        c = np.interp(e[k], np.arange(7), cum)
        assert abs(c - 100 * k / 4) < 1e-9


def _halo_select_ref(x, lo, hi, w):
    xi = x[:, 0]
    return np.nonzero(xi - lo < w)[0], np.nonzero(hi - xi < w)[0]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = slab.DistTransport(rank, world)
        # exchange: message matching with a duplicate neighbour and an empty message
        a = torch.full((rank + 1, 2), float(rank))
        b = torch.zeros((0, 2))
        r_lo, r_hi = tr.exchange(a, b)
        p = workloads.tiny(11, n=2500, clump_frac=0.3, n_dup=4)
        h = p.h0.astype(np.float64) * 1.3
        edges = [0.0, 0.47, 1.0]
        lo, hi = edges[rank], edges[rank + 1]
        own = np.nonzero((p.x[:, 0] >= lo) & (p.x[:, 0] < hi))[0]
        w = float(h.max()) * 1.0001
        ilo, ihi = _halo_select_ref(p.x[own], lo, hi, w)
        if world == 2:
            ihi = np.setdiff1d(ihi, ilo)
        cols = lambda idx: torch.from_numpy(np.ascontiguousarray(own[idx][:, None].astype(np.float64)))
        g_lo, g_hi = tr.exchange(cols(ilo), cols(ihi))
        halo = np.concatenate([g_lo.numpy()[:, 0], g_hi.numpy()[:, 0]]).astype(np.int64)
        local = np.concatenate([own, halo])
        assert len(np.unique(local)) == len(local), "a particle arrived twice"
        x = p.x[local].astype(np.float64)
        den = oracle.density_at(x, p.v[local], p.m[local], h[local], p.box, targets=np.arange(own.size))
        q.put((rank, r_lo.numpy().copy(), r_hi.numpy().copy(), own, den["rho"], den["n_nbr"]))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_and_halo_completeness():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # each rank sent `a` to its lower neighbour: with two ranks the peer is also its upper
    # neighbour, so `a` arrives as "from upper"; the empty "to upper" message arrives as an
    # empty "from lower"
    for r in range(world):
        other = 1 - r
        assert res[r][2].shape == (other + 1, 2) and np.all(res[r][2] == other)
        assert res[r][1].shape == (0, 2)
    # owned results equal the whole-box oracle
    p = workloads.tiny(11, n=2500, clump_frac=0.3, n_dup=4)
    h = p.h0.astype(np.float64) * 1.3
    ref = oracle.density_at(p.x, p.v, p.m, h, p.box)
    seen = np.zeros(p.n, dtype=int)
    for r in range(world):
        own, rho, nn = res[r][3], res[r][4], res[r][5]
        seen[own] += 1
        assert np.allclose(rho, ref["rho"][own], rtol=1e-13)
        assert np.array_equal(nn, ref["n_nbr"][own])
    assert np.all(seen == 1)
