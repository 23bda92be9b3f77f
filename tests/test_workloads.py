"""Input generators: determinism, the fp32 2^-24 grid, config shapes."""
import numpy as np
import pytest

import workloads


def test_deterministic_and_quantised():
    a = workloads.c1()
    b = workloads.c1()
    assert np.array_equal(a.x, b.x) and np.array_equal(a.v, b.v)
    assert a.x.dtype == np.float32 and a.x.shape == (32768, 3)
    k = a.x.astype(np.float64) * (1 << 24)
    assert np.array_equal(k, np.floor(k))
    assert a.x.min() >= 0 and a.x.max() < 1


def test_config_shapes():
    c2 = workloads.c2()
    assert c2.n == 64 ** 3 and np.all(c2.v == 0)
    c3 = workloads.c3()
    assert c3.n == 96 ** 3 + 48 ** 3 and c3.box == (2.0, 1.0, 1.0)
    left = c3.x[:, 0] < 1.0
    # rho_L = 1 (m * 96^3 in unit volume), rho_R = 0.125
    assert abs(c3.m[0] * left.sum() - 1.0) < 1e-5
    assert abs(c3.m[0] * (~left).sum() - 0.125) < 1e-5
    assert set(np.unique(c3.u).tolist()) == {2.5, 2.0}


@pytest.mark.slow
def test_c4_counts():
    p = workloads.c4()
    assert p.n == 2097152
    assert np.all(p.h0 == 0) and p.x.max() < 1.0
    assert p.meta["n_clumps"] == 64
