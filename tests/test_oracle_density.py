"""Pins for oracle.sph: N(h), the h root, density, Omega, div/curl.

Pinned against: the isolated-particle closed form; perfect-lattice closed forms
(re-derived here independently from exact integer shell sums with
mpmath, no neighbour search); the Omega identity (algebra, Appendix A7);
finite differences; linear-velocity-field closed forms (A9); a pure-Python
double-loop brute force on a tiny unequal-mass input.
"""
import math

import mpmath
import numpy as np
import pytest

import oracle
import workloads
from oracle import kernel as K
from oracle.neighbours import min_image

mpmath.mp.dps = 30


def _f_mp(q):
    if q <= 0.5:
        return 1 - 6 * q ** 2 + 6 * q ** 3
    if q <= 1:
        return 2 * (1 - q) ** 3
    return mpmath.mpf(0)


def _fp_mp(q):
    if q <= 0.5:
        return -12 * q + 18 * q ** 2
    if q <= 1:
        return -6 * (1 - q) ** 2
    return mpmath.mpf(0)


def _shells(kind):
    """{squared distance in lattice units: multiplicity}; unit = Delta (SC) or
    Delta_bar = (V/N)^(1/3) (FCC)."""
    sh = {}
    R = 5
    for i in range(-R, R + 1):
        for j in range(-R, R + 1):
            for k in range(-R, R + 1):
                if kind == "FCC" and (i + j + k) % 2:
                    continue
                s = i * i + j * j + k * k
                sh[s] = sh.get(s, 0) + 1
    if kind == "FCC":          # points (i,j,k)*a/2 with a = 4^(1/3) Delta_bar
        scale = (mpmath.mpf(4) ** (mpmath.mpf(1) / 3) / 2) ** 2
        return {mpmath.mpf(s) * scale: c for s, c in sh.items()}
    return {mpmath.mpf(s): c for s, c in sh.items()}


def _lattice_closed_form(kind):
    sh = _shells(kind)

    def N(hh):
        return mpmath.mpf(32) / 3 * sum(c * _f_mp(mpmath.sqrt(s) / hh) for s, c in sh.items())

    hh = mpmath.findroot(lambda t: N(t) - 48, (mpmath.mpf(2.2), mpmath.mpf(2.3)),
                         solver="anderson")
    rho = 8 / mpmath.pi / hh ** 3 * sum(c * _f_mp(mpmath.sqrt(s) / hh) for s, c in sh.items())
    sum_qfp = sum(c * (mpmath.sqrt(s) / hh) * _fp_mp(mpmath.sqrt(s) / hh) for s, c in sh.items())
    omega = -(8 / mpmath.pi / hh ** 3) / (3 * rho) * sum_qfp
    nn = sum(c for s, c in sh.items() if 0 < mpmath.sqrt(s) < hh)
    return float(hh), float(rho), float(omega), nn


@pytest.mark.parametrize("kind", ["SC", "FCC"])
def test_closed_forms_rederived(kind, gold):
    g = gold("lattice_closed_forms.txt")
    hh, rho, om, nn = _lattice_closed_form(kind)
    assert hh == pytest.approx(g[f"{kind}_h_over_delta"], rel=1e-13)
    assert rho == pytest.approx(g[f"{kind}_rho_delta3_over_m"], rel=1e-13)
    assert om == pytest.approx(g[f"{kind}_omega"], rel=1e-11)
    assert nn == g[f"{kind}_n_nbr"]


@pytest.mark.parametrize("kind", ["SC", "FCC"])
def test_oracle_on_perfect_lattice(kind, gold):
    g = gold("lattice_closed_forms.txt")
    p = workloads.c2_exact(k=16) if kind == "SC" else workloads.fcc_exact(k=16)
    d = p.meta["spacing"]
    x = p.x.astype(np.float64)
    h = oracle.solve_h(x, p.box)
    assert np.allclose(h / d, g[f"{kind}_h_over_delta"], rtol=1e-12, atol=0)
    den = oracle.density_at(x, p.v, p.m, h, p.box)
    m = float(p.m[0])
    assert np.allclose(den["rho"] * d ** 3 / m, g[f"{kind}_rho_delta3_over_m"], rtol=1e-12)
    assert np.allclose(den["omega"], g[f"{kind}_omega"], rtol=1e-10)
    assert np.all(den["n_nbr"] == g[f"{kind}_n_nbr"])
    assert np.allclose(den["N"], 48.0, rtol=1e-12)
    assert np.all(den["n_borderline"] == 0)


def test_isolated_particle():
    """One particle with no neighbour inside h: rho = 8m/(pi h^3), Omega = 0, N = 32/3."""
    x = np.array([[0.5, 0.5, 0.5], [0.9, 0.1, 0.1]])
    v = np.zeros((2, 3))
    m = np.array([2.0, 3.0])
    h = np.array([0.1, 0.1])
    d = oracle.density_at(x, v, m, h, (1, 1, 1))
    assert d["rho"][0] == pytest.approx(8 * 2.0 / (math.pi * 0.1 ** 3), rel=1e-14)
    assert abs(d["omega"][0]) < 1e-14
    assert d["N"][0] == pytest.approx(32 / 3, rel=1e-15)
    assert d["n_nbr"][0] == 0


def _tiny_with_h(t=0, n=500):
    p = workloads.tiny(t, n=n)
    return p, p.x.astype(np.float64), p.h0.astype(np.float64)


def test_omega_identity_and_dn_dh():
    p, x, h = _tiny_with_h(1)
    d = oracle.density_at(x, p.v, p.m, h, p.box)
    assert np.allclose(d["omega"], d["omega_identity"], rtol=1e-11, atol=1e-12)
    # dN/dh by finite differences of N(h) (Eq. 3), on particles away from the band
    eps = 1e-7
    dp = oracle.density_at(x, p.v, p.m, h * (1 + eps), p.box)["N"]
    dm = oracle.density_at(x, p.v, p.m, h * (1 - eps), p.box)["N"]
    fd = (dp - dm) / (2 * eps * h)
    ok = d["n_borderline"] == 0
    assert np.allclose(d["dN_dh"][ok], fd[ok], rtol=1e-5, atol=1e-6 / h[ok])
    # d rho/dh likewise
    rp = oracle.density_at(x, p.v, p.m, h * (1 + eps), p.box)["rho"]
    rm = oracle.density_at(x, p.v, p.m, h * (1 - eps), p.box)["rho"]
    fdr = (rp - rm) / (2 * eps * h)
    assert np.allclose(d["drho_dh"][ok], fdr[ok], rtol=1e-5, atol=1e-6 * np.abs(fdr[ok]).max())


def test_density_brute_force_loops():
    """Pure-Python double loop over all pairs (independent of the tree and of
    numpy indexing), unequal masses, h spanning 100x, wrap-around clump."""
    p = workloads.tiny(2, n=120)
    x = p.x.astype(np.float64)
    v = p.v.astype(np.float64)
    m = p.m.astype(np.float64)
    h = p.h0.astype(np.float64) * 2.0
    L = 1.0
    d = oracle.density_at(x, v, m, h, p.box)
    for i in range(0, 120, 7):
        rho = 0.0
        div = 0.0
        curl = [0.0, 0.0, 0.0]
        cnt = 0
        for j in range(120):
            dx = []
            for k in range(3):
                t = x[i, k] - x[j, k]
                if t > L / 2:
                    t -= L
                if t < -L / 2:
                    t += L
                dx.append(t)
            r = math.sqrt(dx[0] ** 2 + dx[1] ** 2 + dx[2] ** 2)
            if r < h[i]:
                q = r / h[i]
                fq = 1 - 6 * q * q + 6 * q ** 3 if q <= 0.5 else 2 * (1 - q) ** 3
                rho += m[j] * 8 / (math.pi * h[i] ** 3) * fq
                if j != i:
                    cnt += 1
                    fp = -12 * q + 18 * q * q if q <= 0.5 else -6 * (1 - q) ** 2
                    dWdr = 8 / (math.pi * h[i] ** 4) * fp
                    gw = [dWdr * dx[k] / r if r > 0 else 0.0 for k in range(3)]
                    dv = [v[j, k] - v[i, k] for k in range(3)]
                    div += m[j] * sum(dv[k] * gw[k] for k in range(3))
                    cr = [dv[1] * gw[2] - dv[2] * gw[1], dv[2] * gw[0] - dv[0] * gw[2],
                          dv[0] * gw[1] - dv[1] * gw[0]]
                    for k in range(3):
                        curl[k] -= m[j] * cr[k]
        assert d["rho"][i] == pytest.approx(rho, rel=1e-13)
        assert d["n_nbr"][i] == cnt
        assert d["div"][i] == pytest.approx(div / rho, rel=1e-10, abs=1e-12)
        assert np.allclose(d["curl"][i], np.array(curl) / rho, rtol=1e-10, atol=1e-12)


def test_h_root_properties():
    p = workloads.tiny(4, n=800, clump_frac=0.3)
    x = p.x.astype(np.float64)
    h = oracle.solve_h(x, p.box)
    d = oracle.density_at(x, p.v, p.m, h, p.box)
    assert np.allclose(d["N"], 48.0, rtol=1e-11)
    # strictly increasing N(h): a slightly smaller h gives fewer, larger gives more
    lo = oracle.density_at(x, p.v, p.m, h * (1 - 1e-6), p.box)["N"]
    hi = oracle.density_at(x, p.v, p.m, h * (1 + 1e-6), p.box)["N"]
    assert np.all(lo < 48.0) and np.all(hi > 48.0)
    # subset solve equals full solve (targets independent of each other)
    sub = np.arange(0, 800, 37)
    assert np.allclose(oracle.solve_h(x, p.box, targets=sub), h[sub], rtol=1e-13)


@pytest.mark.parametrize("field", ["expansion", "rotation"])
def test_linear_velocity_field_on_lattice(field, gold):
    """div(s x) = 3 s Omega and curl(w x x) = 2 w Omega on a perfect SC lattice
    (SURVEY A9), on targets more than h from the wrap."""
    g = gold("lattice_closed_forms.txt")
    p = workloads.c2_exact(k=16)
    x = p.x.astype(np.float64)
    c = np.array([0.5, 0.5, 0.5])
    if field == "expansion":
        v = 0.7 * (x - c)
    else:
        v = np.cross(np.array([0.0, 0.0, 0.3]), x - c)
    h = np.full(p.n, g["SC_h_over_delta"] / 16)
    inner = np.nonzero(np.all(np.abs(x - c) < 0.25, axis=1))[0]
    d = oracle.density_at(x, v, p.m, h, p.box, targets=inner)
    if field == "expansion":
        assert np.allclose(d["div"], g["SC_div_expansion_s0p7"], rtol=1e-9)
        assert np.allclose(d["curl"], 0.0, atol=1e-10)
    else:
        assert np.allclose(d["curl"][:, 2], g["SC_curlz_rotation_w0p3"], rtol=1e-6)
        assert np.allclose(d["curl"][:, :2], 0.0, atol=1e-10)
        assert np.allclose(d["div"], 0.0, atol=1e-10)


def test_galilean_invariance_of_div_curl():
    p, x, h = _tiny_with_h(5)
    d0 = oracle.density_at(x, p.v, p.m, h, p.box)
    d1 = oracle.density_at(x, p.v.astype(np.float64) + np.array([3.0, -2.0, 1.0]), p.m, h, p.box)
    assert np.allclose(d0["div"], d1["div"], rtol=1e-9, atol=1e-9)
    assert np.allclose(d0["curl"], d1["curl"], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("t", [0, 1])
def test_div_curl_bounded_by_their_scale(t):
    """|div_i| <= S_dv,i and |curl_i| <= S_dv,i (Cauchy-Schwarz on each term), with equality
    impossible to exceed by more than rounding; S_dv = 0 only without a neighbour at r > 0."""
    p = workloads.tiny(t, n=500)
    h = p.h0.astype(np.float64) * 1.5
    d = oracle.density_at(p.x, p.v, p.m, h, p.box)
    assert np.all(np.abs(d["div"]) <= d["S_dv"] * (1 + 1e-12))
    assert np.all(np.linalg.norm(d["curl"], axis=1) <= d["S_dv"] * (1 + 1e-12))
    # S_dv = 0 only where particle i has no neighbour at r > 0 inside h_i
    assert np.all((d["S_dv"] > 0) | (d["n_nbr"] - d["n_coincident"] == 0))