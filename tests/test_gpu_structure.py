"""Structure tests of the neighbour-finding machinery (SURVEY §4 layer 2), read back through
sph_debug_export: the sort's permutation, the target groups, the 13 presorted directions of
the leaves and the interaction lists against the brute-force pair set. These
check the intermediate structures directly, not only the sums computed from them (the
paper's correctness rests on its conflict handling; here on these invariants)."""
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


def _run(p, **cfg):
    import torch

    import paper_1404_2303_b200 as sph
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ctx = sph.Context(sph.default_config(p.box, **cfg))
    ctx.build_cells(t(p.x))
    d = ctx.density(t(p.v), t(p.m), t(p.u))
    ctx.force(t(p.v))
    ex = {k: ctx.export(k) for k in ("perm", "groups", "list_off", "list_len", "list", "nodes", "sortoff",
                                     "sorted", "xh")}
    ex["h"] = d.h.cpu().numpy()
    ctx.close()
    return ex


def _tiny():
    p = workloads.tiny(21, n=2500, clump_frac=0.4, n_dup=3)
    p.h0[:] = 0.0
    return p


@pytest.mark.parametrize("cfg", [dict(split_count=48, split_fraction=0.0),
                                 dict(split_count=300, split_fraction=0.875, sort_min_len=0)])
def test_permutation_groups_and_cell_order(cfg):
    p = _tiny()
    ex = _run(p, **cfg)
    n = p.n
    perm = ex["perm"].astype(np.int64)
    assert np.array_equal(np.sort(perm), np.arange(n))                  # a permutation
    assert np.array_equal(ex["xh"][:, :3], p.x[perm])                    # exact copies in cell order
    g = ex["groups"]
    first, cnt = g[:, 1].astype(np.int64), g[:, 2].astype(np.int64)
    assert np.all((cnt >= 1) & (cnt <= 32))
    cover = np.zeros(n, np.int64)
    for a, c in zip(first, cnt):
        cover[a:a + c] += 1
    assert np.all(cover == 1)                                            # groups partition the particles
    # every node's particles are a contiguous cell-order range nested in its parent's
    nodes = ex["nodes"]
    for nd in range(nodes.shape[0]):
        f, c, ch, mask = nodes[nd]
        if ch >= 0:
            kids = [ch + k for k in range(bin(mask & 0xff).count("1"))]
            assert sum(nodes[k][1] for k in kids) == c
            assert nodes[kids[0]][0] == f


def test_presorted_lists_are_sorted_permutations():
    """sort_min_len = 0 (every leaf presorted): each leaf holds 13 lists, each a permutation of
    the leaf's particles in ascending order of the projection on its direction; key differences
    equal the differences of the projected positions."""
    p = _tiny()
    ex = _run(p, split_count=300, split_fraction=0.875, sort_min_len=0)
    nodes, off, srt, xh = ex["nodes"], ex["sortoff"], ex["sorted"], ex["xh"]
    dirs = []
    for k in range(14, 27):
        d = np.array([k // 9 - 1, (k // 3) % 3 - 1, k % 3 - 1], np.float64)
        dirs.append(d / np.linalg.norm(d))
    checked = 0
    for nd in np.nonzero(off >= 0)[0]:
        f, c = int(nodes[nd][0]), int(nodes[nd][1])
        for d in range(13):
            e = srt[off[nd] + d * c: off[nd] + (d + 1) * c]
            assert np.array_equal(np.sort(e["idx"]), np.arange(f, f + c))
            assert np.all(np.diff(e["key"]) >= 0)
            proj = xh[e["idx"], :3].astype(np.float64) @ dirs[d]
            assert np.allclose(e["key"] - e["key"][0], proj - proj[0], atol=4e-7)
            checked += 1
    assert checked >= 13


@pytest.mark.parametrize("cfg", [dict(split_count=48, split_fraction=0.0),
                                 dict(split_count=300, split_fraction=0.875, sort_min_len=0)])
def test_interaction_lists_cover_the_brute_force_pairs(cfg):
    """Every pair with r < max(h_i, h_j) (brute force, fp64 minimum image, the borderline band
    included) appears in the target's group list with the periodic image that realises the
    minimum image; no list holds a (source, image) entry twice."""
    p = _tiny()
    ex = _run(p, **cfg)
    n = p.n
    L = np.asarray(p.box, np.float64)
    xh = ex["xh"].astype(np.float64)
    h = ex["h"][ex["perm"].astype(np.int64)].astype(np.float64)          # cell order
    g = ex["groups"]
    owner = np.empty(n, np.int64)
    for k, (nd, f, c, _) in enumerate(g):
        owner[f:f + c] = k
    lists = []
    for k in range(g.shape[0]):
        e = ex["list"][ex["list_off"][k]: ex["list_off"][k] + ex["list_len"][k]]
        j = (e & ((1 << 27) - 1)).astype(np.int64)
        code = (e >> 27).astype(np.int64)
        key = j * 27 + code
        assert np.unique(key).size == key.size
        lists.append(set(key.tolist()))
    shifts = np.array([[(-L[0] if c % 3 == 1 else L[0] if c % 3 == 2 else 0.0),
                        (-L[1] if (c // 3) % 3 == 1 else L[1] if (c // 3) % 3 == 2 else 0.0),
                        (-L[2] if c // 9 == 1 else L[2] if c // 9 == 2 else 0.0)] for c in range(27)])
    missing = 0
    total = 0
    for s in range(n):
        dx = xh[s, :3] - xh[:, :3]
        dxm = dx - L * np.round(dx / L)
        r = np.sqrt((dxm * dxm).sum(1))
        near = np.nonzero(r < np.maximum(h[s], h) * (1 + 2e-6))[0]
        for j in near:
            if j == s:
                continue
            total += 1
            # the image code whose shift realises the minimum image of source j
            img = np.argmin(np.abs((xh[s, :3] - (xh[j, :3] + shifts)) - dxm[j]).sum(1))
            if j * 27 + img not in lists[owner[s]]:
                missing += 1
    assert total > 10 * n
    assert missing == 0, (missing, total)
