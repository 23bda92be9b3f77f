"""Parity helpers: run the CUDA path through the C ABI, then compare with the oracle
on the same seeded inputs (SURVEY §8(c) comparison modes, north_star tolerances).

  mode A (end to end): GPU h vs the oracle's own root of Eq. 3: rel <= 1e-5.
  mode B (given h):   the oracle evaluated at the GPU's fp32 h (promoted):
      rho rel <= 1e-5;  n_nbr / n_nbr_force exact except |n_gpu - n_or| <= borderline
      pairs (|r/h - 1| <= 1e-6); |da_i| <= 1e-4 S_a,i and |ddu_i| <= 1e-4 S_u,i with the
      per-particle magnitude scales S of SURVEY O8; |dOmega| <= 1e-4 max(1, |Omega|);
      |ddiv_i|, |dcurl_i| <= 1e-4 S_dv,i with the div/curl magnitude scale
      S_dv,i = (1/rho_i) sum_j m_j |v_j - v_i| |grad W_ij| (oracle.density_at; the same
      construction as S_a, reading R25); v_sig rel <= 1e-5.
"""
from __future__ import annotations

import numpy as np

import oracle

TOL_H = 1e-5
TOL_RHO = 1e-5
TOL_FORCE = 1e-4


def run_gpu(p, device_arrays=True, **cfg):
    import torch

    import paper_1404_2303_b200 as sph

    cfg.setdefault("n_ngb_tol", 1e-4)
    ctx = sph.Context(sph.default_config(p.box, **cfg))
    if device_arrays:
        dev = torch.device("cuda:0")
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        x, v, m, u, h0 = t(p.x), t(p.v), t(p.m), t(p.u), t(p.h0)
    else:
        x, v, m, u, h0 = p.x, p.v, p.m, p.u, p.h0
    has_h0 = bool(np.any(p.h0 > 0))
    ctx.build_cells(x, h0 if has_h0 else None)
    d = ctx.density(v, m, u)
    f = ctx.force(v)
    out = {}
    for k in ("h", "rho", "omega", "n_nbr", "div", "curl"):
        a = getattr(d, k)
        out[k] = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    for k in ("a", "dudt", "vsig", "n_nbr_force"):
        a = getattr(f, k)
        out[k] = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    out["stats_density"] = d.stats
    out["stats_force"] = f.stats
    out["launches"] = ctx.kernel_launches
    ctx.close()
    return out


def oracle_given_h(p, h, targets=None):
    """Oracle (mode B) at the GPU's h for `targets` (all if None). Neighbour state for the
    force comes from the oracle's own density at the GPU h of those neighbours."""
    x = p.x.astype(np.float64)
    v = p.v.astype(np.float64)
    m = p.m.astype(np.float64)
    u = p.u.astype(np.float64)
    h = np.asarray(h, dtype=np.float64)
    n = x.shape[0]
    if targets is None:
        targets = np.arange(n)
    targets = np.asarray(targets)
    ci, j, _, _ = oracle.sph.force_pairs(x, h, p.box, targets)
    J = np.unique(np.concatenate([targets, j]))
    den = oracle.density_at(x, v, m, h, p.box, targets=J)
    st = oracle.particle_state(den["rho"], den["omega"], u[J], h[J], den["div"], den["curl"])
    full = {k: np.full(n, np.nan) for k in ("rho", "A", "c", "f")}
    full["rho"][J] = den["rho"]
    full["A"][J] = st["A"]
    full["c"][J] = st["c"]
    full["f"][J] = st["f"]
    fo = oracle.force_at(x, v, m, h, full["rho"], full["A"], full["c"], full["f"], p.box, targets=targets)
    pos = np.searchsorted(J, targets)
    res = {k: (val[pos] if isinstance(val, np.ndarray) and val.shape[:1] == (J.size,) else val)
           for k, val in den.items()}
    res.update({k: st[k][pos] for k in st})
    fo = dict(fo)
    fo["n_borderline_force"] = fo.pop("n_borderline")
    res.update(fo)
    res["targets"] = targets
    return res


def compare(gpu, orc, targets, check_force=True):
    """Assert the north_star tolerances; return a summary dict."""
    t = targets
    rep = {}
    rel_rho = np.abs(gpu["rho"][t] - orc["rho"]) / orc["rho"]
    rep["rho_rel_max"] = float(rel_rho.max())
    assert rep["rho_rel_max"] <= TOL_RHO, rep
    dn = np.abs(gpu["n_nbr"][t].astype(np.int64) - orc["n_nbr"])
    assert np.all(dn <= orc["n_borderline"]), ("n_nbr", int(dn.max()))
    rep["n_nbr_mismatch"] = int((dn > 0).sum())
    om_err = np.abs(gpu["omega"][t] - orc["omega"])
    rep["omega_abs_max"] = float(om_err.max())
    assert rep["omega_abs_max"] <= 1e-4 * max(1.0, float(np.abs(orc["omega"]).max()))
    # div/curl against their per-particle magnitude scale S_dv (|div|, |curl| <= S_dv)
    ddiv = np.abs(gpu["div"][t] - orc["div"])
    dcurl = np.linalg.norm(gpu["curl"][t] - orc["curl"], axis=1)
    sdv = orc["S_dv"]
    with np.errstate(divide="ignore", invalid="ignore"):
        rep["div_rel_max"] = float(np.max(np.where(sdv > 0, ddiv / sdv, np.where(ddiv > 0, np.inf, 0.0))))
        rep["curl_rel_max"] = float(np.max(np.where(sdv > 0, dcurl / sdv, np.where(dcurl > 0, np.inf, 0.0))))
    assert rep["div_rel_max"] <= TOL_FORCE and rep["curl_rel_max"] <= TOL_FORCE, rep
    if check_force:
        ea = np.linalg.norm(gpu["a"][t] - orc["a"], axis=1) / orc["S_a"]
        eu = np.abs(gpu["dudt"][t] - orc["dudt"]) / np.maximum(orc["S_u"], 1e-300)
        rep["a_rel_scale_max"] = float(ea.max())
        rep["du_rel_scale_max"] = float(eu[orc["S_u"] > 0].max()) if np.any(orc["S_u"] > 0) else 0.0
        assert rep["a_rel_scale_max"] <= TOL_FORCE, rep
        assert rep["du_rel_scale_max"] <= TOL_FORCE, rep
        dnf = np.abs(gpu["n_nbr_force"][t].astype(np.int64) - orc["n_nbr_force"])
        assert np.all(dnf <= orc["n_borderline_force"]), ("n_nbr_force", int(dnf.max()))
        rep["vsig_rel_max"] = float((np.abs(gpu["vsig"][t] - orc["vsig"]) / orc["vsig"]).max())
        assert rep["vsig_rel_max"] <= 1e-5, rep
    return rep
