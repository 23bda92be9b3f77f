"""fp64 oracle of the SPH density and force evaluation (TEST INFRASTRUCTURE).

Gather form: every target particle i sums over its own neighbour set, written
out as in the paper (no cells, no sorting, no symmetric tricks). Readings of
the paper that this file takes are marked R<n>.

  Eq. 2  rho_i   = sum_{r_ij < h_i} m_j W(r_ij, h_i)   self term included (R2)
  Eq. 3  N_i(h)  = (4 pi/3) h^3 sum_j W(r_ij, h) = (32/3) sum_j f(r_ij/h)
  P:183-185           h_i solves N_i(h_i) = N_ngb (unique root, R3/R4)
  P:198-199           Omega_i = 1 + h_i/(3 rho_i) d rho_i/d h
  P:198, P:201        P_i = (gamma-1) rho_i u_i,  c_i = sqrt(gamma P_i/rho_i)  (R11)
  Eq. 4  a_i     = -sum_{r_ij < max(h_i,h_j)} m_j [A_i gradW(h_i) + A_j gradW(h_j)]
  Eq. 5      du_i/dt = A_i sum_{r_ij < h_i} m_j v_ij . gradW(h_i)           (R14)
  P:1291-1313         Monaghan-Balsara viscosity (1/4 and 1/8 prefactors), Balsara f_i
                      with the c_i/h_i reading of the denominator (R10), div/curl (R15)

with A_i = P_i/(Omega_i rho_i^2), gradW(h) = G(r,h) dx_ij, dx_ij = x_i - x_j (R12).
"""
from __future__ import annotations

import dataclasses

import numpy as np
from scipy.spatial import cKDTree

from . import kernel as K
from .neighbours import ball_pairs, knn_sorted_distances, min_image

BAND = 1e-6          # borderline band |r/h - 1| <= 1e-6 (north_star; R5)


@dataclasses.dataclass
class OracleConfig:
    gamma: float = 5.0 / 3.0
    n_ngb: float = 48.0
    alpha: float = 0.8
    balsara_eps: float = 1e-4


def _f64(a):
    return np.asarray(a, dtype=np.float64)


# ----------------------------------------------------------------- Eq. 3 --------
def n_ngb_of_h(d, h):
    """N(h) = (32/3) sum_j f(d_j/h) over distances d (self = 0 included); Eq. 3."""
    d = _f64(d)
    h = _f64(h)
    return (32.0 / 3.0) * K.f(d / h[..., None]).sum(axis=-1)


def dn_dh(d, h):
    """dN/dh = -(32/3)/h sum_j q_j f'(q_j)  (>= 0)."""
    d = _f64(d)
    h = _f64(h)
    q = d / h[..., None]
    return -(32.0 / 3.0) / h * (q * K.fprime(q)).sum(axis=-1)


def _root_on_sorted(D, n_t, lo, hi, max_iter=200):
    """Safeguarded Newton/bisection for N(h) = n_t on cached sorted distances D[T,K].
    Requires N(lo) < n_t <= N(hi). Returns h (fp64)."""
    lo = lo.copy()
    hi = hi.copy()
    h = hi.copy()
    active = np.ones(h.shape, dtype=bool)
    for _ in range(max_iter):
        if not active.any():
            break
        a = np.nonzero(active)[0]
        Na = n_ngb_of_h(D[a], h[a])
        dNa = dn_dh(D[a], h[a])
        res = Na - n_t
        below = res < 0
        lo[a] = np.where(below, h[a], lo[a])
        hi[a] = np.where(below, hi[a], h[a])
        done = (np.abs(res) <= 1e-13 * n_t) | ((hi[a] - lo[a]) <= 2e-16 * hi[a])
        with np.errstate(divide="ignore", invalid="ignore"):
            hn = h[a] - res / dNa
        bad = ~np.isfinite(hn) | (hn <= lo[a]) | (hn >= hi[a])
        hn = np.where(bad, 0.5 * (lo[a] + hi[a]), hn)
        h[a] = np.where(done, h[a], hn)
        active[a] = ~done
    return h


def solve_h(x, box, targets=None, n_ngb=48.0, k0=64, tree=None):
    """h_i := the unique root of N_i(h) = n_ngb.

    N_i(h) = 32/3 for h below the nearest-neighbour distance and strictly
    increasing afterwards, so the root is unique for n_ngb > 32/3. Distances
    come from a k-nearest query (k doubled until N(d_k) >= n_ngb, which
    guarantees every neighbour inside the root is among the k).
    """
    x = _f64(x)
    box = _f64(box)
    if n_ngb <= 32.0 / 3.0:
        raise ValueError("n_ngb must exceed the self term 32/3")
    if targets is None:
        targets = np.arange(x.shape[0])
    targets = np.asarray(targets)
    if tree is None:
        tree = cKDTree(x, boxsize=box)
    h = np.full(targets.shape[0], np.nan)
    todo = np.arange(targets.shape[0])
    k = k0
    while todo.size:
        if k > x.shape[0]:
            raise ValueError("not enough particles for the neighbour target")
        D = knn_sorted_distances(x, box, x[targets[todo]], k, tree=tree)
        dk = D[:, -1] * (1.0 - 1e-12)
        ok = n_ngb_of_h(D, dk) >= n_ngb
        if ok.any():
            idx = np.nonzero(ok)[0]
            lo = np.full(idx.size, 1e-300)
            h[todo[idx]] = _root_on_sorted(D[idx], n_ngb, lo, dk[idx])
        todo = todo[~ok]
        k *= 2
    if np.any(h >= 0.5 * box.min()):
        raise ValueError("solved h >= L/2: too few particles for the periodic box")
    return h


# ----------------------------------------------------------------- Eq. 2 --------
def density_at(x, v, m, h, box, targets=None, tree=None):
    """rho, d rho/dh, Omega, N, dN/dh, n_nbr, div v, curl v at GIVEN h.

    Sums over N_i(h_i) = {j : r_ij < h_i} including j = i (R2, R5 strict '<').
    div_i  =  (1/rho_i) sum_j m_j (v_j - v_i) . gradW(r_ij, h_i)
    curl_i = -(1/rho_i) sum_j m_j (v_j - v_i) x gradW(r_ij, h_i)
    Also returns the Omega identity  -(1/(3 rho_i)) sum_j m_j r_ij dW/dr  (Appendix A7)
    and the borderline / coincident counts (O8).
    """
    x = _f64(x)
    v = _f64(v)
    m = _f64(m)
    h = _f64(h)
    box = _f64(box)
    if targets is None:
        targets = np.arange(x.shape[0])
    targets = np.asarray(targets)
    T = targets.shape[0]
    hi = h[targets]
    ci, j, dx, r = ball_pairs(x, box, x[targets], hi * (1.0 + 2 * BAND), tree=tree)
    border = np.abs(r / hi[ci] - 1.0) <= BAND
    n_border = np.bincount(ci, weights=border & (j != targets[ci]), minlength=T).astype(np.int64)
    keep = r < hi[ci]
    ci, j, dx, r = ci[keep], j[keep], dx[keep], r[keep]
    i = targets[ci]
    hp = hi[ci]
    q = r / hp
    w = K.W(r, hp)
    mj = m[j]

    def S(wts, comp=None):
        return np.bincount(ci, weights=wts, minlength=T)

    rho = S(mj * w)
    drho_dh = S(mj * K.dW_dh(r, hp))
    omega = 1.0 + hi / (3.0 * rho) * drho_dh
    omega_identity = -S(mj * r * K.dW_dr(r, hp)) / (3.0 * rho)
    N = (32.0 / 3.0) * S(K.f(q))
    dN = -(32.0 / 3.0) / hi * S(q * K.fprime(q))
    n_nbr = np.bincount(ci, minlength=T).astype(np.int64) - 1       # minus the self term
    n_coinc = np.bincount(ci, weights=(r == 0) & (j != i), minlength=T).astype(np.int64)
    G = K.grad_scalar(r, hp)
    gradW = G[:, None] * dx                                           # grad_i W(r_ij, h_i)
    dv = v[j] - v[i]                                                  # v_j - v_i
    div = S(mj * np.einsum("ij,ij->i", dv, gradW)) / rho
    cr = np.cross(dv, gradW)
    curl = -np.stack([S(mj * cr[:, k]) for k in range(3)], axis=1) / rho[:, None]
    # magnitude scale of the div / curl sums (O8, like S_a): (1/rho_i) sum_j m_j |v_j - v_i|
    # |grad W|, so that |div_i| <= S_dv,i and |curl_i| <= S_dv,i (Cauchy-Schwarz)
    S_dv = S(mj * np.linalg.norm(dv, axis=1) * np.abs(G) * r) / rho
    return dict(rho=rho, drho_dh=drho_dh, omega=omega, omega_identity=omega_identity,
                N=N, dN_dh=dN, n_nbr=n_nbr, div=div, curl=curl, S_dv=S_dv,
                n_borderline=n_border, n_coincident=n_coinc)


# ----------------------------------------------------------------- ghost --------
def particle_state(rho, omega, u, h, div, curl, cfg: OracleConfig = OracleConfig()):
    """P, c, A = P/(Omega rho^2), Balsara f."""
    rho, omega, u, h, div = map(_f64, (rho, omega, u, h, div))
    curl = _f64(curl)
    g = cfg.gamma
    P = (g - 1.0) * rho * u
    c = np.sqrt(g * P / rho)
    with np.errstate(divide="ignore"):
        A = P / (omega * rho * rho)          # inf for an isolated particle (Omega = 0, R17)
    cn = np.sqrt((curl * curl).sum(axis=-1))
    fb = cn / (np.abs(div) + cn + cfg.balsara_eps * c / h)            # R10: c_i/h_i
    return dict(P=P, c=c, A=A, f=fb)


# ----------------------------------------------------------------- Eq. 4/5 ------
def force_pairs(x, h, box, targets, tree=None):
    """Directed pairs (t, j), j != i = targets[t], with r_ij < max(h_i,h_j)*(1+2e-6).

    The set {j : r < h_i} comes from a ball query around i; {j : r < h_j} from a
    ball query of radius h_j around every particle j against a tree of the
    targets. Their union is the force set."""
    x = _f64(x)
    h = _f64(h)
    box = _f64(box)
    targets = np.asarray(targets)
    T = targets.shape[0]
    ext = 1.0 + 2 * BAND
    c1, j1, _, _ = ball_pairs(x, box, x[targets], h[targets] * ext, tree=tree)
    ttree = cKDTree(x[targets], boxsize=box)
    j2, c2, _, _ = ball_pairs(x[targets], box, x, h * ext, tree=ttree)
    key = np.unique(np.concatenate([c1 * x.shape[0] + j1, c2 * x.shape[0] + j2]))
    ci = key // x.shape[0]
    j = key % x.shape[0]
    keep = j != targets[ci]
    ci, j = ci[keep], j[keep]
    dx = min_image(x[targets[ci]] - x[j], box)
    r = np.sqrt(np.einsum("ij,ij->i", dx, dx))
    return ci, j, dx, r


def force_at(x, v, m, h, rho, A, c, fbal, box, targets=None, alpha=0.8, tree=None):
    """Accelerations, du/dt, v_sig and magnitude scales for the targets.

    State arrays (h, rho, A, c, fbal) are per particle over ALL particles.
    For each j != i with r_ij < max(h_i, h_j):
      G_i = G(r,h_i) (0 if r >= h_i), G_j = G(r,h_j) (0 if r >= h_j)
      w   = min(0, v_ij . dx / r)  (0 at r = 0, R13)
      Pi  = -alpha (c_i + c_j - 3 w) w / (rho_i + rho_j)
      a_i   -= m_j [A_i G_i + A_j G_j + 1/4 Pi (f_i+f_j)(G_i+G_j)] dx
      du_i  += m_j (v_ij . dx) [A_i G_i + 1/8 Pi (f_i+f_j)(G_i+G_j)]
      vsig_i = max_j (c_i + c_j - 3 w)
    """
    x, v, m, h, rho, A, c, fbal = map(_f64, (x, v, m, h, rho, A, c, fbal))
    box = _f64(box)
    if targets is None:
        targets = np.arange(x.shape[0])
    targets = np.asarray(targets)
    T = targets.shape[0]
    ci, j, dx, r = force_pairs(x, h, box, targets, tree=tree)
    i = targets[ci]
    hmax = np.maximum(h[i], h[j])
    border = np.abs(r / hmax - 1.0) <= BAND
    n_border = np.bincount(ci, weights=border, minlength=T).astype(np.int64)
    keep = r < hmax
    ci, j, dx, r, i = ci[keep], j[keep], dx[keep], r[keep], i[keep]
    Gi = np.where(r < h[i], K.grad_scalar(r, h[i]), 0.0)
    Gj = np.where(r < h[j], K.grad_scalar(r, h[j]), 0.0)
    # A_k enters only multiplied by G_k; a particle with no neighbour inside its
    # own h has Omega = 0 (A infinite) but G_k = 0 on every pair: the product is 0.
    with np.errstate(invalid="ignore"):
        AGi = np.where(Gi != 0.0, A[i] * Gi, 0.0)
        AGj = np.where(Gj != 0.0, A[j] * Gj, 0.0)
    vij = v[i] - v[j]
    vdx = np.einsum("ij,ij->i", vij, dx)
    with np.errstate(divide="ignore", invalid="ignore"):
        w = np.where(r > 0, np.minimum(0.0, vdx / np.where(r > 0, r, 1.0)), 0.0)
    Pi = -alpha * (c[i] + c[j] - 3.0 * w) * w / (rho[i] + rho[j])
    V = Pi * (fbal[i] + fbal[j]) * (Gi + Gj)
    Tij = AGi + AGj + 0.25 * V
    mj = m[j]
    a = -np.stack([np.bincount(ci, weights=mj * Tij * dx[:, k], minlength=T)
                   for k in range(3)], axis=1)
    du = np.bincount(ci, weights=mj * vdx * (AGi + 0.125 * V), minlength=T)
    vsig = np.zeros(T)
    np.maximum.at(vsig, ci, c[i] + c[j] - 3.0 * w)
    S_a = np.bincount(ci, weights=mj * np.abs(Tij) * r, minlength=T)
    S_u = np.bincount(ci, weights=mj * np.abs(vdx) * (np.abs(AGi) + 0.125 * np.abs(V)),
                      minlength=T)
    n_nbr = np.bincount(ci, minlength=T).astype(np.int64)
    du_visc = np.bincount(ci, weights=mj * vdx * 0.125 * V, minlength=T)
    return dict(a=a, dudt=du, vsig=vsig, S_a=S_a, S_u=S_u, n_nbr_force=n_nbr,
                n_borderline=n_border, dudt_visc=du_visc,
                n_pairs_directed=int(ci.size))


# ----------------------------------------------------------------- pipeline -----
def evaluate_all(x, v, m, u, box, h=None, cfg: OracleConfig = OracleConfig()):
    """Whole evaluation for every particle: h (own root unless given), density,
    particle state, force. Returns a dict of fp64 arrays + pair counts."""
    x = _f64(x)
    box = _f64(box)
    tree = cKDTree(x, boxsize=box)
    if h is None:
        h = solve_h(x, box, n_ngb=cfg.n_ngb, tree=tree)
    h = _f64(h)
    d = density_at(x, v, m, h, box, tree=tree)
    st = particle_state(d["rho"], d["omega"], u, h, d["div"], d["curl"], cfg)
    fo = force_at(x, v, m, h, d["rho"], st["A"], st["c"], st["f"], box,
                  alpha=cfg.alpha, tree=tree)
    out = dict(h=h)
    out.update(d)
    out.update(st)
    out.update(fo)
    out["n_pairs"] = fo["n_pairs_directed"] // 2          # F (unordered)
    out["n_directed"] = int(d["n_nbr"].sum())             # D
    return out
