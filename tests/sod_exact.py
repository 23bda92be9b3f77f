"""Exact solution of the Riemann problem for an ideal gas (Sod 1978, the paper's Sod-shock
test), used to validate the time-stepped SPH system. Test
infrastructure only. This is the textbook construction restated: the star-region pressure
p* solves f_L(p) + f_R(p) + (u_R - u_L) = 0 with
  f_K(p) = (p - p_K) sqrt(A_K / (p + B_K)),  A_K = 2 / ((gamma+1) rho_K), B_K = (gamma-1)/(gamma+1) p_K
for a shock (p > p_K) and
  f_K(p) = 2 c_K / (gamma-1) ((p / p_K)^((gamma-1)/(2 gamma)) - 1)
for a rarefaction (p <= p_K); u* = (u_L + u_R)/2 + (f_R(p*) - f_L(p*))/2; the density on
each side of the contact follows the shock (Rankine-Hugoniot) or isentropic relations, and
the solution is self-similar in xi = x / t."""
import numpy as np


def _f(p, rho, pk, ck, g):
    if p > pk:
        A = 2.0 / ((g + 1) * rho)
        B = (g - 1) / (g + 1) * pk
        val = (p - pk) * np.sqrt(A / (p + B))
        der = np.sqrt(A / (B + p)) * (1 - (p - pk) / (2 * (B + p)))
    else:
        val = 2 * ck / (g - 1) * ((p / pk) ** ((g - 1) / (2 * g)) - 1)
        der = (p / pk) ** (-(g + 1) / (2 * g)) / (rho * ck)
    return val, der


def star_state(rl, ul, pl, rr, ur, pr, g):
    cl, cr = np.sqrt(g * pl / rl), np.sqrt(g * pr / rr)
    p = 0.5 * (pl + pr)
    for _ in range(100):
        fl, dl = _f(p, rl, pl, cl, g)
        fr, dr = _f(p, rr, pr, cr, g)
        dp = (fl + fr + ur - ul) / (dl + dr)
        p = max(p - dp, 1e-12)
        if abs(dp) < 1e-14 * p:
            break
    fl, _ = _f(p, rl, pl, cl, g)
    fr, _ = _f(p, rr, pr, cr, g)
    return p, 0.5 * (ul + ur) + 0.5 * (fr - fl)


def density(xi, rl, ul, pl, rr, ur, pr, g=5.0 / 3.0):
    """rho(xi = x/t) of the Riemann problem (left state for xi -> -inf)."""
    xi = np.asarray(xi, dtype=np.float64)
    ps, us = star_state(rl, ul, pl, rr, ur, pr, g)
    cl, cr = np.sqrt(g * pl / rl), np.sqrt(g * pr / rr)
    out = np.empty_like(xi)
    gm = (g - 1) / (g + 1)
    # left wave
    if ps > pl:   # shock
        rs_l = rl * (ps / pl + gm) / (gm * ps / pl + 1)
        sl = ul - cl * np.sqrt((g + 1) / (2 * g) * ps / pl + (g - 1) / (2 * g))
        left = np.where(xi < sl, rl, rs_l)
    else:         # rarefaction
        rs_l = rl * (ps / pl) ** (1 / g)
        cs_l = cl * (ps / pl) ** ((g - 1) / (2 * g))
        head, tail = ul - cl, us - cs_l
        fan = rl * np.maximum(2 / (g + 1) + (g - 1) / ((g + 1) * cl) * (ul - xi), 0.0) ** (2 / (g - 1))
        left = np.where(xi < head, rl, np.where(xi < tail, fan, rs_l))
    # right wave
    if ps > pr:   # shock
        rs_r = rr * (ps / pr + gm) / (gm * ps / pr + 1)
        sr = ur + cr * np.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
        right = np.where(xi > sr, rr, rs_r)
    else:
        rs_r = rr * (ps / pr) ** (1 / g)
        cs_r = cr * (ps / pr) ** ((g - 1) / (2 * g))
        head, tail = ur + cr, us + cs_r
        fan = rr * np.maximum(2 / (g + 1) - (g - 1) / ((g + 1) * cr) * (ur - xi), 0.0) ** (2 / (g - 1))
        right = np.where(xi > head, rr, np.where(xi > tail, fan, rs_r))
    out[:] = np.where(xi < us, left, right)
    return out
