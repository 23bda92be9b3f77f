"""Periodic neighbour search for the oracle (TEST INFRASTRUCTURE).

Geometry (periodic domain P:482-484): dx_ij = x_i - x_j per
component, minimum image (subtract L if dx > L/2, add L if dx < -L/2), exact
in fp64 for fp32 inputs; r_ij = |dx_ij|. Requires every search radius < L/2.

`ball_pairs` uses scipy's cKDTree (a library primitive) only to enumerate
candidates; membership is then decided here, in fp64, from the min-image dx
(strict r < radius). `brute_pairs` is the O(N*T) definition, used by the tests
to pin `ball_pairs`.
"""
from __future__ import annotations

import itertools

import numpy as np
from scipy.spatial import cKDTree

#: threads of the cKDTree queries (-1 = all; a process pool sets 1 per process)
WORKERS = -1


def min_image(dx: np.ndarray, box) -> np.ndarray:
    box = np.asarray(box, dtype=np.float64)
    dx = np.array(dx, dtype=np.float64, copy=True)
    dx = np.where(dx > 0.5 * box, dx - box, dx)
    dx = np.where(dx < -0.5 * box, dx + box, dx)
    return dx


def _finish(x, box, ci, j, centers_x, radii):
    dx = min_image(centers_x[ci] - x[j], box)
    r = np.sqrt(np.einsum("ij,ij->i", dx, dx))
    keep = r < radii[ci]
    return ci[keep], j[keep], dx[keep], r[keep]


def ball_pairs(x, box, centers_x, radii, tree=None, chunk=200_000):
    """All (c, j) with r(centers_x[c], x[j]) < radii[c] (strict), periodic.

    Returns (ci, j, dx, r) with dx = centers_x[c] - x[j] (min image). Pairs are
    ordered by c, then ascending j.
    """
    x = np.asarray(x, dtype=np.float64)
    centers_x = np.asarray(centers_x, dtype=np.float64).reshape(-1, 3)
    radii = np.broadcast_to(np.asarray(radii, dtype=np.float64), (centers_x.shape[0],))
    box = np.asarray(box, dtype=np.float64)
    assert np.all(radii < 0.5 * box.min()), "search radius must be < L/2 (min image)"
    if tree is None:
        tree = cKDTree(x, boxsize=box)
    out = []
    for s in range(0, centers_x.shape[0], chunk):
        cx = centers_x[s:s + chunk]
        rr = radii[s:s + chunk]
        # candidate superset: the tree's own distance may differ from ours by an ulp
        lists = tree.query_ball_point(cx, rr * (1.0 + 1e-9) + 1e-300, workers=WORKERS,
                                      return_sorted=True)
        lens = np.fromiter(map(len, lists), dtype=np.int64, count=len(lists))
        j = np.fromiter(itertools.chain.from_iterable(lists), dtype=np.int64,
                        count=int(lens.sum()))
        ci = np.repeat(np.arange(s, s + cx.shape[0], dtype=np.int64), lens)
        out.append(_finish(x, box, ci, j, centers_x, radii))
    ci, j, dx, r = (np.concatenate(z) for z in zip(*out)) if out else (
        np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 3)), np.zeros(0))
    return ci, j, dx, r


def brute_pairs(x, box, centers_x, radii):
    """O(N*T) definition of ball_pairs (used to pin it)."""
    x = np.asarray(x, dtype=np.float64)
    centers_x = np.asarray(centers_x, dtype=np.float64).reshape(-1, 3)
    radii = np.broadcast_to(np.asarray(radii, dtype=np.float64), (centers_x.shape[0],))
    cis, js, dxs, rs = [], [], [], []
    for c in range(centers_x.shape[0]):
        dx = min_image(centers_x[c][None, :] - x, box)
        r = np.sqrt((dx * dx).sum(axis=1))
        jj = np.nonzero(r < radii[c])[0]
        cis.append(np.full(jj.size, c, dtype=np.int64))
        js.append(jj.astype(np.int64))
        dxs.append(dx[jj])
        rs.append(r[jj])
    return (np.concatenate(cis), np.concatenate(js), np.concatenate(dxs).reshape(-1, 3),
            np.concatenate(rs))


def knn_sorted_distances(x, box, centers_x, k, tree=None):
    """Distances (fp64, min image, recomputed here) of the k nearest particles to
    each centre, ascending, the centre itself included when it is a particle."""
    x = np.asarray(x, dtype=np.float64)
    centers_x = np.asarray(centers_x, dtype=np.float64).reshape(-1, 3)
    if tree is None:
        tree = cKDTree(x, boxsize=np.asarray(box, dtype=np.float64))
    k = min(k, x.shape[0])
    _, idx = tree.query(centers_x, k=k, workers=WORKERS)
    idx = idx.reshape(centers_x.shape[0], k)
    dx = min_image(centers_x[:, None, :] - x[idx], box)
    d = np.sqrt((dx * dx).sum(axis=2))
    return np.sort(d, axis=1)
