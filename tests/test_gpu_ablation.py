"""The paper's cell-pair loops (sph_pair_ablation): naive and sorted sweeps
give the hot path's density, find the same pairs, and on uniform random points in cells of edge
h their window-pass and in-range rates are the paper's (P:624-629 with reading R9: face 50.0 %
window / 33.5 % in range; edge 16.2 % / 9.2 %; corner 3.6 % / 2.1 %; SURVEY A5 Monte Carlo)."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests must run on the B200 box")
    from paper_1404_2303_b200 import build
    build.build()


def _ctx(p, h0=None, **cfg):
    import torch

    import paper_1404_2303_b200 as sph
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ctx = sph.Context(sph.default_config(p.box, **cfg))
    ctx.build_cells(t(p.x), None if h0 is None else t(h0))
    d = ctx.density(t(p.v), t(p.m), t(p.u))
    return ctx, d


@pytest.mark.parametrize("name", ["C1", "tiny"])
def test_naive_and_sorted_match_the_hot_path(name):
    import torch
    p = workloads.c1() if name == "C1" else workloads.tiny(2, n=4000, clump_frac=0.3, n_dup=0)
    if name == "tiny":
        p.h0[:] = 0.0
    ctx, d = _ctx(p, split_count=48, split_fraction=0.0)
    out = {}
    for s in (False, True):
        rho = torch.empty_like(d.rho)
        c = ctx.pair_ablation(s, rho)
        out[s] = c
        assert float(((rho - d.rho).abs() / d.rho).max()) <= 1e-5
        assert c["hits"] == d.stats["n_directed"]          # every directed contribution, once
    assert out[True]["tests"] < out[False]["tests"]
    ctx.close()


def _expected_counts(x, h, nc):
    """fp64 brute force over the 13 forward neighbour classes of a periodic nc^3 grid: particle
    pairs, sweep-1 window passes (r_j + shift <= r_i + h_i along the canonical direction) and
    pairs within h_i, by class (face, edge, corner)."""
    x = x.astype(np.float64)
    cell = np.floor(x.astype(np.float32) * np.float32(nc)).astype(np.int64) % nc
    cid = (cell[:, 2] * nc + cell[:, 1]) * nc + cell[:, 0]
    order = np.argsort(cid, kind="stable")
    starts = np.searchsorted(cid[order], np.arange(nc ** 3 + 1))
    E = 1.0 / nc
    out = np.zeros((3, 3), np.int64)   # [class][pairs, pass, inrange]
    for k in range(14, 27):
        o = np.array([k // 9 - 1, (k // 3) % 3 - 1, k % 3 - 1])
        u = o / np.linalg.norm(o)
        cls = int(np.count_nonzero(o)) - 1
        for ca in range(nc ** 3):
            a = np.array([ca % nc, (ca // nc) % nc, ca // (nc * nc)])
            b = (a + o) % nc
            cb = (b[2] * nc + b[1]) * nc + b[0]
            A = order[starts[ca]:starts[ca + 1]]
            Bp = order[starts[cb]:starts[cb + 1]]
            if A.size == 0 or Bp.size == 0:
                continue
            ra = (x[A] - a * E) @ u
            rb = (x[Bp] - b * E) @ u + (o * E) @ u
            dxv = x[A][:, None, :] - (x[Bp][None, :, :] + (a + o - b)[None, None, :] * E)
            r = np.sqrt((dxv ** 2).sum(-1))
            hi = h[A][:, None]
            out[cls, 0] += A.size * Bp.size
            out[cls, 1] += int((rb[None, :] <= ra[:, None] + hi).sum())
            out[cls, 2] += int((r < hi).sum())
    return out


def test_window_pass_and_in_range_counts():
    """uniform random points (C1's) with h near the cell edge (h0 = edge, margin 1): the
    sweep-1 window passes and in-range pairs per neighbour class equal an fp64 brute force, and
    the rates are the paper's (R9) up to the spread of h about the edge."""
    p = workloads.c1()
    nc = 16
    h0 = np.full(p.n, (1.0 / nc) * (1 - 2e-5), np.float32)
    ctx, d = _ctx(p, h0=h0, n_ngb_tol=1e9, h_margin=1.0, split_count=48, split_fraction=0.0)
    h = d.h.cpu().numpy().astype(np.float64)
    c = ctx.pair_ablation(True)
    assert c["cells_x"] == nc
    exp = _expected_counts(p.x, h, nc)
    for cls, name in enumerate(("face", "edge", "corner")):
        assert c["pairs_" + name] == exp[cls, 0]
        assert abs(c["pass_" + name] - exp[cls, 1]) <= 10, (name, c["pass_" + name], exp[cls, 1])
        assert abs(c["inrange_" + name] - exp[cls, 2]) <= 10, (name, c["inrange_" + name], exp[cls, 2])
    hr = float(np.median(h)) * nc     # h / edge
    paper = {"face": (0.500, 0.335), "edge": (0.162, 0.092), "corner": (0.036, 0.021)}
    for name, (pw, pr) in paper.items():
        w = c["pass_" + name] / c["pairs_" + name]
        ir = c["inrange_" + name] / c["pairs_" + name]
        assert w == pytest.approx(pw, rel=0.15 + 3 * abs(hr - 1)), (name, w, hr)
        assert ir == pytest.approx(pr, rel=0.15 + 3 * abs(hr - 1)), (name, ir, hr)
    ctx.close()
