"""Multi-rank host protocol of the slab decomposition on the CPU (gloo, world sizes 2 and 3):
the band re-send when an owned h outgrows the halo, the re-partition (`migrate`) and the
work-weighted cuts (`partition`). The device work is played by `FakeCtx`, which answers the
same calls from the fp64 oracle (tests only), so the exchanges, message order and the halo
bookkeeping are what is checked here; tests/test_gpu_slab.py runs the same code on libsph.
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
from paper_1404_2303_b200.sph import SPH_E_NOCONV, SphError


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _D:
    pass


class FakeCtx:
    """The libsph calls slab.py makes, answered on the CPU (oracle h and rho, fp64)."""

    def __init__(self, box, lo, hi, width):
        self.box, self.lo, self.hi, self.width = box, lo, hi, width
        self.need = 0.0
        self.imported = None

    def halo_select(self, x, lo, hi, width):
        xi = x[:, 0]
        return (torch.nonzero(xi - lo < width)[:, 0].to(torch.int32),
                torch.nonzero(hi - xi < width)[:, 0].to(torch.int32))

    def slab_leavers(self, x, lo, hi):
        xi = x[:, 0]
        return torch.nonzero(xi < lo)[:, 0].to(torch.int32), torch.nonzero(xi >= hi)[:, 0].to(torch.int32)

    def x_histogram(self, x, lo, hi, nbins):
        b = torch.clamp(((x[:, 0].double() - lo) / (hi - lo) * nbins).floor().long(), 0, nbins - 1)
        return torch.bincount(b, minlength=nbins).to(torch.int64)

    def x_histogram_weighted(self, x, w, lo, hi, nbins):
        b = torch.clamp(((x[:, 0].double() - lo) / (hi - lo) * nbins).floor().long(), 0, nbins - 1)
        return torch.bincount(b, weights=w.double(), minlength=nbins).round().to(torch.int64)

    def set_halo_width(self, w):
        self.width = w

    def halo_required(self):
        return self.need

    def build_cells_halo(self, X, n_own, H0):
        self.X, self.n_own = X.numpy().astype(np.float64), n_own

    def density(self, V, M, U):
        n = self.n_own
        h = oracle.solve_h(self.X, self.box, targets=np.arange(n))
        xi = self.X[:n, 0]
        near = (xi - self.lo < h) | (self.hi - xi < h)
        self.need = float(h[near].max()) if near.any() else 0.0
        if self.need > self.width:
            raise SphError(SPH_E_NOCONV, "halo too narrow")
        hh = np.zeros(self.X.shape[0])
        hh[:n] = h
        den = oracle.density_at(self.X, V.numpy(), M.numpy(), hh, self.box, targets=np.arange(n))
        self.h = h
        d = _D()
        d.h, d.rho, d.n_nbr, d.stats = torch.from_numpy(h), torch.from_numpy(den["rho"]), None, {}
        return d

    def export_state(self, idx):
        out = torch.zeros(int(idx.shape[0]), 5, dtype=torch.float64)
        out[:, 0] = torch.from_numpy(self.h[idx.long().numpy()])
        return out

    def import_halo_state(self, state):
        self.imported = state.clone()

    def force(self, like):
        f = _D()
        f.a = f.dudt = f.n_nbr_force = None
        f.stats = {}
        return f


def _band_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = workloads.tiny(31, n=2400, clump_frac=0.35, n_dup=0)
        edges = [k / world for k in range(world + 1)]
        lo, hi = edges[rank], edges[rank + 1]
        own = np.nonzero((p.x[:, 0] >= lo) & (p.x[:, 0] < hi))[0]
        width0 = 0.02                      # far below the largest h near a face: band rounds needed
        ctx = FakeCtx(p.box, lo, hi, width0)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).astype(np.float64))
        tr = slab.DistTransport(rank, world)
        r = slab.evaluate_rank(ctx, t(p.x[own]), t(p.v[own]), t(p.m[own]), t(p.u[own]), t(p.h0[own]), lo, hi,
                               width0, tr)
        halo_x = ctx.X[ctx.n_own:]
        q.put((rank, own, r.h.numpy(), r.rho.numpy(), halo_x, ctx.imported[:, 0].numpy(), ctx.width))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world, *extra):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q) + extra) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_band_resend_reproduces_the_whole_box(world):
    """A halo 0.02 wide (the clumps' outskirts need h ~ 0.1): the first density fails on some
    rank, every rank sends the missing band and evaluates again; owned h and rho equal the
    whole-box oracle, and the halo state imported before the force (first rows + band rows,
    in the order of the received halo) is the global h of exactly those particles."""
    res = _spawn(_band_worker, world)
    p = workloads.tiny(31, n=2400, clump_frac=0.35, n_dup=0)
    x = p.x.astype(np.float64)
    h = oracle.solve_h(x, p.box)
    ref = oracle.density_at(x, p.v, p.m, h, p.box)
    pos = {tuple(r): i for i, r in enumerate(x)}
    seen = np.zeros(p.n, int)
    for rank in range(world):
        _, own, hr, rho, halo_x, imp_h, width = res[rank]
        seen[own] += 1
        assert width > 0.02                                  # a band round happened
        assert np.allclose(hr, h[own], rtol=1e-12)
        assert np.allclose(rho, ref["rho"][own], rtol=1e-12)
        ids = np.array([pos[tuple(r)] for r in halo_x])
        assert len(np.unique(ids)) == len(ids)               # no particle arrived twice
        assert not np.isin(ids, own).any()
        assert np.allclose(imp_h, h[ids], rtol=1e-12)
    assert np.all(seen == 1)


def _migrate_worker(rank, world, port, q, shift):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = workloads.tiny(32, n=3000, clump_frac=0.4, n_dup=0)
        tr = slab.DistTransport(rank, world)
        edges = [k / world for k in range(world + 1)]
        own = np.nonzero((p.x[:, 0] >= edges[rank]) & (p.x[:, 0] < edges[rank + 1]))[0]
        ctx = FakeCtx(p.box, edges[rank], edges[rank + 1], 0.1)
        x = torch.from_numpy(p.x[own].astype(np.float32))
        w = torch.from_numpy((1 + own % 7).astype(np.int32))          # work units
        # weighted cuts: quantiles of the global weighted histogram
        cuts = slab.partition(ctx, tr, x, 0.0, 1.0, world, w=w, nbins=4096)
        cuts_n = slab.partition(ctx, tr, x, 0.0, 1.0, world, nbins=4096)
        new = list(cuts)
        new[1:-1] = [c + shift for c in new[1:-1]]
        arrays = {"x": x, "v": torch.from_numpy(p.v[own]), "id": torch.from_numpy(own.astype(np.int32)), "w": w}
        out = slab.migrate(ctx, tr, new[rank], new[rank + 1], arrays)
        q.put((rank, cuts, cuts_n, new, {k: v.numpy() for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shift", [(2, 0.013), (3, -0.021)])
def test_partition_and_migrate(world, shift):
    res = _spawn(_migrate_worker, world, shift)
    p = workloads.tiny(32, n=3000, clump_frac=0.4, n_dup=0)
    wall = (1 + np.arange(p.n) % 7).astype(np.float64)
    # the weighted cuts split the total work at k / world (linear inside a 1/4096 bin)
    cuts = res[0][1]
    order = np.argsort(p.x[:, 0])
    cw = np.cumsum(wall[order])
    for k in range(1, world):
        below = wall[p.x[:, 0] < cuts[k]].sum()
        assert abs(below - cw[-1] * k / world) <= 1e-2 * cw[-1], (k, below, cw[-1] * k / world)
    assert res[0][2] != cuts                                  # counts and work give other cuts
    ids = []
    for rank in range(world):
        _, c, _, new, out = res[rank]
        assert c == cuts                                      # every rank computed the same cuts
        xs = out["x"][:, 0]
        assert np.all((xs >= new[rank]) & (xs < new[rank + 1]))
        i = out["id"].astype(np.int64)
        assert np.array_equal(out["x"], p.x[i])               # rows travelled whole
        assert np.array_equal(out["v"], p.v[i])
        assert np.array_equal(out["w"], (1 + i % 7).astype(np.int32))
        ids.append(i)
    ids = np.concatenate(ids)
    assert np.array_equal(np.sort(ids), np.arange(p.n))
