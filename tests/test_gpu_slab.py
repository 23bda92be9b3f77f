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
