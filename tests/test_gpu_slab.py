"""Slab decomposition on ONE GPU: P ranks evaluated one after another in one process (no
rank ever waits on another), halo buffers passed directly; the owned results must equal
the single-context evaluation (and therefore the oracle) within the parity tolerances."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [2, 3, 4])
def test_slabs_match_single_context(P):
    import torch

    import paper_1404_2303_b200 as sph
    from paper_1404_2303_b200 import slab
    from tests import parity

    p = workloads.c1()
    ref = parity.run_gpu(p)
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    h0 = np.full(p.n, 0.0704508, dtype=np.float32)
    width = 0.12                                   # > max h (0.09) with margin
    edges = [k / P for k in range(P + 1)]
    ranks, owns = [], []
    for r in range(P):
        own = np.nonzero((p.x[:, 0] >= edges[r]) & (p.x[:, 0] < edges[r + 1]))[0]
        owns.append(own)
        cfg = sph.default_config(p.box, rank=r, nranks=P, slab_lo=edges[r], slab_hi=edges[r + 1], halo_width=width)
        ctx = sph.Context(cfg)
        ranks.append(slab.SlabRank(ctx, t(p.x[own]), t(p.v[own]), t(p.m[own]), t(p.u[own]), t(h0[own]),
                                   edges[r], edges[r + 1], width, P))
    out = slab.evaluate_ring_sequential(ranks)
    for r in range(P):
        own = owns[r]
        o = out[r]
        assert o.n_halo > 0
        h = o.h.cpu().numpy()
        assert np.allclose(h, ref["h"][own], rtol=2e-6)
        assert np.allclose(o.rho.cpu().numpy(), ref["rho"][own], rtol=1e-5)
        assert np.array_equal(o.n_nbr.cpu().numpy(), ref["n_nbr"][own])
        assert np.array_equal(o.n_nbr_force.cpu().numpy(), ref["n_nbr_force"][own])
        a = o.a.cpu().numpy()
        scale = np.abs(ref["a"]).max()
        assert np.abs(a - ref["a"][own]).max() <= 1e-4 * scale
    for rk in ranks:
        rk.ctx.close()


def test_halo_pack_kernel_equals_the_row_layout():
    """sph_halo_pack (k_halo_pack) writes exactly the rows slab.pack builds: {x, v, m, u, h0} of
    the selected owned particles."""
    import torch

    import paper_1404_2303_b200 as sph
    from paper_1404_2303_b200 import slab

    p = workloads.tiny(1, n=3000)
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = sph.Context(sph.default_config(p.box))
    x, v, m, u, h0 = t(p.x), t(p.v), t(p.m), t(p.u), t(p.h0)
    lo_idx, hi_idx = ctx.halo_select(x, 0.25, 0.75, 0.1)
    assert lo_idx.numel() > 0 and hi_idx.numel() > 0
    ref = slab.pack(x, v, m, u, h0)
    for idx in (lo_idx, hi_idx):
        assert torch.equal(ctx.halo_pack(x, v, m, u, h0, idx), ref[idx.long()])
    ctx.close()


def test_band_resend_with_a_narrow_halo():
    """Halo width 0.03 on C1 (max h ~0.09): the first density fails on the ranks whose owned
    particles near a face need more, every rank sends the band up to the required width
    (sph_halo_required, k_hface) and evaluates again; results equal the single context."""
    import torch

    import paper_1404_2303_b200 as sph
    from paper_1404_2303_b200 import slab
    from tests import parity

    p = workloads.c1()
    ref = parity.run_gpu(p)
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    P, width = 3, 0.03
    h0 = np.full(p.n, 0.0704508, dtype=np.float32)
    edges = [k / P for k in range(P + 1)]
    ranks, owns = [], []
    for r in range(P):
        own = np.nonzero((p.x[:, 0] >= edges[r]) & (p.x[:, 0] < edges[r + 1]))[0]
        owns.append(own)
        cfg = sph.default_config(p.box, rank=r, nranks=P, slab_lo=edges[r], slab_hi=edges[r + 1], halo_width=width)
        ranks.append(slab.SlabRank(sph.Context(cfg), t(p.x[own]), t(p.v[own]), t(p.m[own]), t(p.u[own]),
                                   t(h0[own]), edges[r], edges[r + 1], width, P))
    out = slab.evaluate_ring_sequential(ranks)
    need = max(rk.ctx.halo_required() for rk in ranks)
    assert ranks[0].width > width and need <= ranks[0].width
    for r in range(P):
        own, o = owns[r], out[r]
        assert np.allclose(o.h.cpu().numpy(), ref["h"][own], rtol=2e-6)
        assert np.allclose(o.rho.cpu().numpy(), ref["rho"][own], rtol=1e-5)
        assert np.array_equal(o.n_nbr_force.cpu().numpy(), ref["n_nbr_force"][own])
        scale = np.abs(ref["a"]).max()
        assert np.abs(o.a.cpu().numpy() - ref["a"][own]).max() <= 1e-4 * scale
    for rk in ranks:
        rk.ctx.close()


def test_leavers_and_weighted_histogram():
    """sph_slab_leavers and sph_x_histogram_weighted against numpy."""
    import torch

    import paper_1404_2303_b200 as sph

    p = workloads.tiny(2, n=5000)
    dev = torch.device("cuda:0")
    ctx = sph.Context(sph.default_config(p.box))
    x = torch.from_numpy(p.x).to(dev)
    lo, hi = 0.3, 0.55
    ilo, ihi = ctx.slab_leavers(x, lo, hi)
    assert np.array_equal(ilo.cpu().numpy(), np.nonzero(p.x[:, 0] < np.float32(lo))[0])
    assert np.array_equal(ihi.cpu().numpy(), np.nonzero(p.x[:, 0] >= np.float32(hi))[0])
    w = (np.arange(p.n) % 11).astype(np.int32)
    hist = ctx.x_histogram_weighted(x, torch.from_numpy(w).to(dev), 0.0, 1.0, 64).cpu().numpy()
    b = np.clip(np.floor((p.x[:, 0] - np.float32(0.0)) / np.float32(1.0) * np.float32(64)).astype(np.int64), 0, 63)
    assert np.array_equal(hist, np.bincount(b, weights=w, minlength=64).astype(np.int64))
    ctx.close()
