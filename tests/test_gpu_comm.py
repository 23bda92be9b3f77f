"""libsph's NCCL transport (include/sph.h sph_comm_*, sph_halo_*, sph_allreduce) on one
GPU: a one-rank communicator, whose lower and upper neighbour are the rank itself, so the
ring exchange must deliver send_hi to recv_lo and send_lo to recv_hi (the message order
the header specifies for nranks <= 2). Multi-rank runs use the same calls; their host
logic is covered by the gloo tests (tests/test_slab_gloo.py)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests must run on the B200 box")
    from paper_1404_2303_b200 import build
    build.build()
    import paper_1404_2303_b200 as sph
    c = sph.Context(sph.default_config((1.0, 1.0, 1.0), rank=0, nranks=1))
    c.comm_init(sph.Context.comm_unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("n_lo,n_hi", [(37, 5), (0, 12), (9, 0), (0, 0)])
def test_self_ring_exchange(ctx, n_lo, n_hi):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n_lo * 100 + n_hi)
    s_lo = torch.rand(n_lo, 9, device="cuda", generator=g)
    s_hi = torch.rand(n_hi, 9, device="cuda", generator=g)
    r_lo, r_hi = ctx.halo_exchange(s_lo, s_hi)
    assert r_lo.shape == s_hi.shape and r_hi.shape == s_lo.shape
    assert torch.equal(r_lo, s_hi) and torch.equal(r_hi, s_lo)


def test_allreduce_one_rank(ctx):
    import torch
    a = torch.tensor([1.5, -2.0, 3.25], dtype=torch.float64, device="cuda")
    b = torch.tensor([7, -1], dtype=torch.int64, device="cuda")
    assert torch.equal(ctx.allreduce_(a.clone(), "sum"), a)
    assert torch.equal(ctx.allreduce_(b.clone(), "max"), b)


def test_lib_transport_interface(ctx):
    """slab.LibTransport (the bench's --transport libsph) on one rank."""
    import torch

    import paper_1404_2303_b200 as sph
    from paper_1404_2303_b200 import slab
    c = sph.Context(sph.default_config((1.0, 1.0, 1.0), rank=0, nranks=1))
    tr = slab.LibTransport(c, 0, 1)
    s_lo, s_hi = torch.rand(4, 5, device="cuda"), torch.rand(6, 5, device="cuda")
    r_lo, r_hi = tr.exchange(s_lo, s_hi)
    assert torch.equal(r_lo, s_hi) and torch.equal(r_hi, s_lo)
    assert tr.allreduce_max(2.5) == 2.5
    h = torch.arange(5, dtype=torch.int64, device="cuda")
    assert torch.equal(tr.allreduce_sum(h.clone()), h)
    c.close()


def test_comm_errors():
    import paper_1404_2303_b200 as sph
    c = sph.Context(sph.default_config((1.0, 1.0, 1.0)))
    import torch
    with pytest.raises(sph.SphError) as e:
        c.halo_exchange(torch.zeros(1, 3, device="cuda"), torch.zeros(1, 3, device="cuda"))
    assert e.value.status == sph.SPH_E_STATE
    c.close()
