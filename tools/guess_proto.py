"""Offline study of cold-start h guesses on C4 (CPU only): how far from the solved h is each
estimator? The spread decides how many particles the NB walk re-walks on a cold start.

  python tools/guess_proto.py [--sample 20000]

E0 reproduces k_guess_h (octree cell occupancy, split_count 48, leaf + ancestors with >= 8
particles up to the first with >= 48). E1.. are candidates that use only the tree's cells.
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (the solved h: the reference this study compares to)
import workloads  # noqa: E402

DEPTH = 12
NNGB = 48.0


def spread3(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def tree(x):
    """cells per level: cell id of every particle at every level, leaf level per particle"""
    q = np.minimum((x * (1 << DEPTH)).astype(np.int64), (1 << DEPTH) - 1)
    key = spread3(q[:, 0]) << np.uint64(2) | spread3(q[:, 1]) << np.uint64(1) | spread3(q[:, 2])
    ids, counts = [], []
    leaf = np.full(x.shape[0], -1, np.int64)
    for l in range(DEPTH + 1):
        cid = (key >> np.uint64(3 * (DEPTH - l))).astype(np.int64)
        u, inv, cnt = np.unique(cid, return_inverse=True, return_counts=True)
        c = cnt[inv]
        ids.append(cid)
        counts.append(c)
        newleaf = (leaf < 0) & (c <= NNGB)
        leaf[newleaf] = l
    leaf[leaf < 0] = DEPTH
    return ids, counts, leaf


def e0(counts, leaf, t):
    """k_guess_h"""
    out = np.empty(t.size)
    for k, i in enumerate(t):
        dens = 0.0
        l = leaf[i]
        while True:
            c = counts[l][i]
            vol = (1.0 / (1 << l)) ** 3
            if c >= 8:
                dens = max(dens, c / vol)
            if c >= NNGB or l == 0:
                if dens == 0.0:
                    dens = c / vol
                break
            l -= 1
        out[k] = (3 * NNGB / (4 * np.pi * dens)) ** (1 / 3)
    return out


def e0_variant(counts, leaf, t, cmin, mode):
    """density of the smallest cell (leaf or ancestor) holding >= cmin particles ("first"),
    or the geometric mean of the densities along the path up to it ("gmean")"""
    out = np.empty(t.size)
    for k, i in enumerate(t):
        l = leaf[i]
        ds = []
        while True:
            c = counts[l][i]
            vol = (1.0 / (1 << l)) ** 3
            if c >= 4:
                ds.append(c / vol)
            if c >= cmin or l == 0:
                if not ds:
                    ds.append(c / vol)
                break
            l -= 1
        dens = ds[-1] if mode == "first" else float(np.exp(np.mean(np.log(ds))))
        out[k] = (3 * (NNGB - 32 / 3) / (4 * np.pi * dens)) ** (1 / 3)
    return out


def leaf_cells(x, ids, counts, leaf):
    """the leaves: (level, integer cell coords, count, tight box lo/hi)"""
    # leaf id = (level, cell id at that level)
    cid = np.empty(x.shape[0], np.int64)
    for l in range(DEPTH + 1):
        m = leaf == l
        cid[m] = ids[l][m]
    pack = leaf.astype(np.int64) * (1 << 40) + cid
    u, inv = np.unique(pack, return_inverse=True)
    nl = u.size
    cnt = np.bincount(inv, minlength=nl)
    lo = np.full((nl, 3), np.inf)
    hi = np.full((nl, 3), -np.inf)
    for d in range(3):
        np.minimum.at(lo[:, d], inv, x[:, d])
        np.maximum.at(hi[:, d], inv, x[:, d])
    lev = (u >> 40).astype(np.int64)
    return inv, lev, cnt, lo, hi


def overlap_1d(a0, a1, b0, b1):
    return np.clip(np.minimum(a1, b1) - np.maximum(a0, b0), 0.0, None)


def e_cube(x, t, inv, lev, cnt, lo, hi, h0, mode, tree_leaves, target=NNGB, shape="cube"):
    """count within a sphere of radius r estimated from leaf boxes (uniform inside each box),
    the sphere replaced by the cube of equal volume; solve count(r) = 48 by bisection"""
    side = (4 * np.pi / 3) ** (1 / 3)   # cube of the sphere's volume: edge = side * r
    if mode == "cell":
        E = 1.0 / (1 << lev)
        centre = (lo + hi) * 0.5
        blo = np.floor(centre / E[:, None]) * E[:, None]
        bhi = blo + E[:, None]
    else:   # tight box, padded to the mean spacing of its particles
        ext = np.maximum(hi - lo, 0.0)
        vol_c = (1.0 / (1 << lev)) ** 3
        pad = 0.5 * (vol_c / np.maximum(cnt, 1)) ** (1 / 3)
        blo = lo - pad[:, None]
        bhi = hi + pad[:, None]
    bvol = np.prod(bhi - blo, axis=1)
    dens = cnt / bvol
    out = np.empty(t.size)
    for k, i in enumerate(t):
        R = 3.0 * h0[k]
        near = tree_leaves.query_ball_point(x[i], R * 1.2)
        near = np.asarray(near, np.int64)
        L = np.unique(inv[near])
        a, b = 0.2 * h0[k], 3.0 * h0[k]
        for _ in range(40):
            r = 0.5 * (a + b)
            if shape == "cube":
                e = 0.5 * side * r
                v = np.ones(L.size)
                for d in range(3):
                    v *= overlap_1d(x[i, d] - e, x[i, d] + e, blo[L, d], bhi[L, d])
            else:   # sphere: the fraction of a 6^3 midpoint grid of each box inside the sphere
                g = (np.arange(6) + 0.5) / 6
                pts = blo[L, None, None, None, :] + (bhi - blo)[L, None, None, None, :] * np.stack(
                    np.meshgrid(g, g, g, indexing="ij"), -1)[None]
                d2 = ((pts - x[i]) ** 2).sum(-1)
                v = (d2 < r * r).mean(axis=(1, 2, 3)) * bvol[L]
            c = float((dens[L] * v).sum())
            if c < target:
                a = r
            else:
                b = r
        out[k] = 0.5 * (a + b)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sample", type=int, default=4000)
    args = ap.parse_args()
    p = workloads.c4()
    x = p.x.astype(np.float64)
    rng = np.random.default_rng(5)
    t = rng.choice(p.n, args.sample, replace=False)
    # keep away from the periodic faces (the prototype has no images)
    t0 = time.time()
    h = oracle.solve_h(p.x, p.box, targets=t)
    print(f"oracle h: {time.time() - t0:.1f} s", flush=True)
    ids, counts, leaf = tree(x)
    g0 = e0(counts, leaf, t)
    inv, lev, cnt, lo, hi = leaf_cells(x, ids, counts, leaf)
    from scipy.spatial import cKDTree
    kt = cKDTree(x)
    res = {"E0 k_guess_h": g0}
    res["E0 k_guess_h, target 48 - 32/3"] = g0 * ((NNGB - 32 / 3) / NNGB) ** (1 / 3)
    for cmin in (16, 48, 96, 192):
        for mode in ("first", "gmean"):
            res[f"E0' {mode} cmin {cmin}"] = e0_variant(counts, leaf, t, cmin, mode)
    res["E1 cube, target 48 - 32/3"] = e_cube(x, t, inv, lev, cnt, lo, hi, g0, "cell", kt, NNGB - 32 / 3)

    inner = np.all((x[t] > 0.1) & (x[t] < 0.9), axis=1)
    for k, g in res.items():
        r = (g / h)[inner]
        qs = np.percentile(r, [1, 10, 50, 90, 99])
        rew = {m: round(float(np.mean(r * m < 1.0)), 3) for m in (1.0, 1.1, 1.2, 1.3)}
        print(f"{k:34s} guess/h p1 {qs[0]:.2f} p10 {qs[1]:.2f} p50 {qs[2]:.2f} p90 {qs[3]:.2f} "
              f"p99 {qs[4]:.2f}  re-walk at margin {rew}  mean (g m)^3 at 1.1 {np.mean((r * 1.1) ** 3):.2f}")


if __name__ == "__main__":
    main()
