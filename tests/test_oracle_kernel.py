"""Pins for oracle/kernel.py against the paper's kernel display
and plain mathematics (normalisation, calculus)."""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import kernel as K


def test_closed_form_values(gold):
    g = gold("kernel_values.txt")
    assert K.W(0.0, 1.0) == pytest.approx(g["W_0"], rel=1e-15)
    assert K.W(0.5, 1.0) == pytest.approx(g["W_half"], rel=1e-15)
    assert K.W(0.75, 1.0) == pytest.approx(g["W_3quarter"], rel=1e-15)
    assert K.W(1.0, 1.0) == g["W_1"]
    assert K.W(1.5, 1.0) == 0.0
    # both branches agree at q = 1/2 (continuity of W and of f')
    assert K.f(0.5) == pytest.approx(2 * 0.5 ** 3, rel=1e-15)
    assert K.fprime(0.5) == pytest.approx(g["fprime_half"], rel=1e-15)
    assert K.fprime(0.5 + 1e-12) == pytest.approx(g["fprime_half"], rel=1e-9)


@pytest.mark.parametrize("h", [0.01, 0.3, 1.0, 7.0])
def test_normalisation(h):
    """int W dV = 1 over the support (a kernel that is not normalised is wrong)."""
    val, err = integrate.quad(lambda r: 4 * math.pi * r * r * float(K.W(r, h)), 0, h,
                              points=[0.5 * h], epsabs=0, epsrel=1e-13)
    assert val == pytest.approx(1.0, rel=1e-11)


def test_derivatives_finite_difference():
    rng = np.random.default_rng(1)
    h = rng.uniform(0.2, 2.0, 200)
    r = h * rng.uniform(0.02, 0.98, 200)
    r = r[np.abs(r / h - 0.5) > 1e-3]
    h = h[: r.size]
    eps = 1e-6
    fd_r = (K.W(r + eps * h, h) - K.W(r - eps * h, h)) / (2 * eps * h)
    fd_h = (K.W(r, h + eps * h) - K.W(r, h - eps * h)) / (2 * eps * h)
    assert np.allclose(K.dW_dr(r, h), fd_r, rtol=1e-7, atol=1e-9 / h ** 4)
    assert np.allclose(K.dW_dh(r, h), fd_h, rtol=1e-7, atol=1e-9 / h ** 4)


def test_grad_scalar():
    q = np.linspace(1e-3, 1.2, 999)
    with np.errstate(divide="ignore"):
        expect = np.where(q <= 1, K.fprime(q) / q, 0.0)
    assert np.allclose(K.g(q), expect, rtol=1e-13, atol=1e-13)
    assert K.g(0.0) == -12.0                                   # finite at r = 0
    # G = dW/dr / r
    r, h = 0.37, 0.8
    assert K.grad_scalar(r, h) == pytest.approx(K.dW_dr(r, h) / r, rel=1e-13)
    assert K.grad_scalar(1.0, 1.0) == 0.0 and K.grad_scalar(1.3, 1.0) == 0.0


def test_monotone_decreasing():
    q = np.linspace(0, 1, 10001)
    fq = K.f(q)
    assert np.all(np.diff(fq) < 0)
    assert fq[0] == 1.0 and fq[-1] == 0.0
