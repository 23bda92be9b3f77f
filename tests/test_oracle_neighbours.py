"""Pin oracle/neighbours.py (cKDTree candidates + fp64 min-image membership)
against the O(N*T) brute-force definition, on inputs with a clump straddling
all periodic boundaries and exact duplicates."""
import numpy as np
import pytest

import workloads
from oracle.neighbours import ball_pairs, brute_pairs, knn_sorted_distances, min_image


def _canon(ci, j, r):
    o = np.lexsort((j, ci))
    return ci[o], j[o], r[o]


@pytest.mark.parametrize("t", [0, 1, 2])
def test_ball_pairs_equals_brute_force(t):
    p = workloads.tiny(t, n=400)
    x = p.x.astype(np.float64)
    radii = p.h0.astype(np.float64)
    a = _canon(*[z for k, z in enumerate(ball_pairs(x, p.box, x, radii)) if k != 2])
    b = _canon(*[z for k, z in enumerate(brute_pairs(x, p.box, x, radii)) if k != 2])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])
    # the corner clump must actually produce wrap-around pairs and coincident pairs
    ci, j, dx, r = ball_pairs(x, p.box, x, radii)
    assert np.any(np.abs(x[ci] - x[j]) > 0.5)
    assert np.any((r == 0) & (ci != j))


def test_min_image_exact_for_fp32_inputs():
    x1 = np.float32(0.99999994)
    x2 = np.float32(5.9604645e-08)
    d = min_image(np.array([[float(x1) - float(x2), 0, 0]]), (1.0, 1.0, 1.0))
    assert d[0, 0] == (float(x1) - 1.0) - float(x2)


def test_knn_matches_brute():
    p = workloads.tiny(3, n=300)
    x = p.x.astype(np.float64)
    D = knn_sorted_distances(x, p.box, x[:20], 40)
    for c in range(20):
        dx = min_image(x[c] - x, p.box)
        r = np.sort(np.sqrt((dx * dx).sum(1)))[:40]
        assert np.allclose(D[c], r, rtol=0, atol=1e-15)
