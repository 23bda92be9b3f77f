"""Cubic-spline smoothing kernel with support radius h (TEST INFRASTRUCTURE).

P:157-166 (section 2.1, the kernel W(r,h) display):

    W(r,h) = 8/(pi h^3) * { 1 - 6 q^2 + 6 q^3      0 <= q <= 1/2
                            2 (1 - q)^3            1/2 < q <= 1
                            0                      q > 1 },   q = r/h.

Derived quantities (plain calculus on that definition, fp64):
    f'(q)      = -12 q + 18 q^2  |  -6 (1-q)^2  |  0
    dW/dr      = 8/(pi h^4) f'(q)
    dW/dh      = -(3 W + r dW/dr) / h
    g(q)       = f'(q)/q = 18 q - 12  |  -6 (1-q)^2 / q  |  0   (finite at q = 0)
    grad_i W(|x_i - x_j|, h) = 8/(pi h^5) g(q) (x_i - x_j)        (reading R12)
"""
from __future__ import annotations

import numpy as np

C_NORM = 8.0 / np.pi


def f(q):
    """Dimensionless spline f(q)."""
    q = np.asarray(q, dtype=np.float64)
    inner = 1.0 - 6.0 * q * q + 6.0 * q * q * q
    outer = 2.0 * (1.0 - q) ** 3
    return np.where(q <= 0.5, inner, np.where(q <= 1.0, outer, 0.0))


def fprime(q):
    """df/dq."""
    q = np.asarray(q, dtype=np.float64)
    inner = -12.0 * q + 18.0 * q * q
    outer = -6.0 * (1.0 - q) ** 2
    return np.where(q <= 0.5, inner, np.where(q <= 1.0, outer, 0.0))


def g(q):
    """f'(q)/q, evaluated without dividing by q on the inner branch (finite at 0)."""
    q = np.asarray(q, dtype=np.float64)
    inner = 18.0 * q - 12.0
    with np.errstate(divide="ignore", invalid="ignore"):
        outer = np.where(q > 0.5, -6.0 * (1.0 - q) ** 2 / np.where(q > 0, q, 1.0), 0.0)
    return np.where(q <= 0.5, inner, np.where(q <= 1.0, outer, 0.0))


def W(r, h):
    """W(r,h) of P:157-166."""
    r = np.asarray(r, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    return C_NORM / h ** 3 * f(r / h)


def dW_dr(r, h):
    r = np.asarray(r, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    return C_NORM / h ** 4 * fprime(r / h)


def dW_dh(r, h):
    r = np.asarray(r, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    return -(3.0 * W(r, h) + r * dW_dr(r, h)) / h


def grad_scalar(r, h):
    """G(r,h) such that grad_i W(|x_i-x_j|, h) = G * (x_i - x_j); G = 8/(pi h^5) g(r/h)."""
    r = np.asarray(r, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    return C_NORM / h ** 5 * g(r / h)
