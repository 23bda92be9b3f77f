"""Pins of the exact Riemann solver (tests/sod_exact.py) against published values of the
classic Sod problem (rho 1 / 0.125, p 1 / 0.1, u 0, gamma 1.4): p* = 0.30313, u* = 0.92745
(the standard reference values of the exact solution), and limits that must hold."""
import numpy as np

from . import sod_exact as S


def test_sod_classic_star_state():
    p, u = S.star_state(1.0, 0.0, 1.0, 0.125, 0.0, 0.1, 1.4)
    assert abs(p - 0.30313) < 1e-5
    assert abs(u - 0.92745) < 1e-5


def test_sod_density_limits_and_plateaus():
    g = 1.4
    xi = np.array([-10.0, 10.0, 0.5, 1.5])
    r = S.density(xi, 1.0, 0.0, 1.0, 0.125, 0.0, 0.1, g)
    assert r[0] == 1.0 and r[1] == 0.125
    # left of the contact (rarefied): rho*_L = rho_L (p*/p_L)^(1/gamma) = 0.42632
    assert abs(r[2] - 0.42632) < 1e-4
    # between contact and shock: rho*_R = 0.26557 (Rankine-Hugoniot)
    assert abs(r[3] - 0.26557) < 1e-4


def test_sod_trivial_and_symmetric():
    r = S.density(np.linspace(-2, 2, 9), 1.0, 0.0, 1.0, 1.0, 0.0, 1.0)
    assert np.allclose(r, 1.0)
    a = S.density(np.array([-0.3, 0.3]), 1.0, 0.0, 1.0, 0.125, 0.0, 0.1)
    b = S.density(np.array([0.3, -0.3]), 0.125, 0.0, 0.1, 1.0, 0.0, 1.0)   # mirrored problem
    assert np.allclose(a, b)
