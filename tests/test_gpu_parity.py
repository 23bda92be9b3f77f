"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs. Tolerances are the north_star's (BASELINE.json), see tests/parity.py."""
import numpy as np
import pytest

import oracle
import workloads

from . import parity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests must run on the B200 box")
    from paper_1404_2303_b200 import build
    build.build()


def _modes(p, targets=None, check_force=True, **cfg):
    g = P.run_gpu(p, **cfg)
    h_or = oracle.solve_h(p.x, p.box, targets=targets)
    t = np.arange(p.n) if targets is None else targets
    rel_h = np.abs(g["h"][t] - h_or) / h_or
    assert rel_h.max() <= P.TOL_H, float(rel_h.max())                 # mode A
    orc = P.oracle_given_h(p, g["h"], targets=t)                       # mode B
    rep = P.compare(g, orc, t, check_force=check_force)
    rep["h_rel_max"] = float(rel_h.max())
    return g, orc, rep


@pytest.mark.parametrize("t", [0, 1, 2])
def test_tiny_clumped_unequal_mass(t):
    """uniform + a Gaussian clump straddling the periodic corner, unequal masses,
    exact duplicates (coincident pairs), h spanning ~10x; all particles compared."""
    p = workloads.tiny(t, n=4000, clump_frac=0.3, n_dup=5)
    p.h0[:] = 0.0                       # library initial guess
    g, orc, rep = _modes(p)
    assert g["stats_density"]["n_unconverged"] == 0
    assert np.all(orc["n_coincident"][np.nonzero(orc["n_coincident"])] > 0)


def test_c1_full():
    p = workloads.c1()
    g, orc, rep = _modes(p)
    st = g["stats_force"]
    # F and D agree with the oracle's counts up to borderline pairs
    assert abs(st["n_pairs"] - orc["n_pairs_directed"] // 2) <= orc["n_borderline_force"].sum()
    assert abs(g["stats_density"]["n_directed"] - orc["n_nbr"].sum()) <= orc["n_borderline"].sum()


def test_c1_host_pointers_equal_device_pointers():
    p = workloads.c1()
    a = P.run_gpu(p, device_arrays=True)
    b = P.run_gpu(p, device_arrays=False)
    for k in ("h", "rho", "a", "dudt", "n_nbr", "n_nbr_force"):
        assert np.array_equal(a[k], b[k]), k                            # deterministic


@pytest.mark.parametrize("kind", ["SC", "FCC"])
def test_perfect_lattice_closed_forms(kind, gold):
    gd = gold("lattice_closed_forms.txt")
    p = workloads.c2_exact(k=32) if kind == "SC" else workloads.fcc_exact(k=32)
    g = P.run_gpu(p)
    d = p.meta["spacing"]
    m = float(p.m[0])
    assert np.allclose(g["h"] / d, gd[f"{kind}_h_over_delta"], rtol=1e-5)
    assert np.allclose(g["rho"] * d ** 3 / m, gd[f"{kind}_rho_delta3_over_m"], rtol=1e-5)
    assert np.allclose(g["omega"], gd[f"{kind}_omega"], rtol=1e-4)
    assert np.all(g["n_nbr"] == gd[f"{kind}_n_nbr"])
    assert np.all(g["n_nbr_force"] == gd[f"{kind}_n_nbr"])
    # at rest on a perfect lattice: zero force by symmetry, du/dt exactly 0
    orc = P.oracle_given_h(p, g["h"], targets=np.arange(0, p.n, 997))
    assert np.all(np.linalg.norm(g["a"], axis=1) <= 1e-5 * orc["S_a"].max())
    assert np.all(g["dudt"] == 0.0)


def test_c2_sampled():
    p = workloads.c2()
    t = workloads.subsample_box(p, 0.01, seed=2)
    _modes(p, targets=t)


def test_c3_sampled_with_interfaces():
    """two resolutions (2x in h) and two periodic density interfaces: sample includes the
    particles closest to x = 0, 1, 2."""
    p = workloads.c3()
    rng = np.random.default_rng(3)
    near = np.nonzero((np.abs(p.x[:, 0] - 1.0) < 0.03) | (p.x[:, 0] < 0.03) | (p.x[:, 0] > 1.97))[0]
    t = np.unique(np.concatenate([rng.choice(p.n, 1500, replace=False), rng.choice(near, 1500, replace=False)]))
    _modes(p, targets=t)


def test_c4_sampled_full_size():
    """the headline workload at full size, in the bench's launch configuration (cold h0)."""
    p = workloads.c4()
    rng = np.random.default_rng(4)
    t = np.sort(rng.choice(p.n, 1500, replace=False))
    g, orc, rep = _modes(p, targets=t)
    assert g["stats_density"]["n_unconverged"] == 0


def test_conservation_c1():
    p = workloads.c1()
    g = P.run_gpu(p)
    m = p.m.astype(np.float64)
    a = g["a"].astype(np.float64)
    mom = np.abs((m[:, None] * a).sum(0)).max() / (m[:, None] * np.abs(a)).sum()
    assert mom < 1e-5
    v = p.v.astype(np.float64)
    e = abs((m * ((v * a).sum(1) + g["dudt"])).sum()) / (m * (np.abs((v * a).sum(1)) + np.abs(g["dudt"]))).sum()
    assert e < 1e-5


def test_permutation_invariance():
    p = workloads.c1()
    rng = np.random.default_rng(9)
    perm = rng.permutation(p.n)
    q = p.take(perm)
    a = P.run_gpu(p)
    b = P.run_gpu(q)
    assert np.allclose(a["h"][perm], b["h"], rtol=2e-6)
    assert np.allclose(a["rho"][perm], b["rho"], rtol=1e-5)
    assert np.array_equal(a["n_nbr"][perm], b["n_nbr"])


def test_errors():
    import torch

    import paper_1404_2303_b200 as sph
    ctx = sph.Context(sph.default_config((1, 1, 1)))
    x = torch.rand(1000, 3, device="cuda")
    v = torch.zeros(1000, 3, device="cuda")
    m = torch.ones(1000, device="cuda")
    u = torch.ones(1000, device="cuda")
    with pytest.raises(sph.SphError) as e:
        ctx.density(v, m, u)
    assert e.value.status == sph.SPH_E_STATE
    bad = x.clone()
    bad[3, 1] = 1.0                                   # x must be < L
    with pytest.raises(sph.SphError) as e:
        ctx.build_cells(bad)
    assert e.value.status == sph.SPH_E_DOMAIN
    with pytest.raises(sph.SphError) as e:
        ctx.build_cells(x, torch.full((1000,), 0.5, device="cuda"))   # h >= L/3
    assert e.value.status == sph.SPH_E_DOMAIN
    ctx.build_cells(x)
    with pytest.raises(sph.SphError) as e:
        ctx.density(v, -m, u)
    assert e.value.status == sph.SPH_E_DOMAIN
    with pytest.raises(sph.SphError) as e:
        ctx.force(v)
    assert e.value.status == sph.SPH_E_STATE
    ctx.close()


def test_paper_mode_membership():
    """n_ngb_tol = 1 (the paper's "e.g. +-1"): several h are correct, so h parity is
    replaced by membership (SURVEY 8(c) "paper" mode): for every particle the oracle's
    N(h_gpu) lies in [47, 49]; then mode B at the GPU's h."""
    p = workloads.tiny(3, n=4000, clump_frac=0.3, n_dup=0)
    p.h0[:] = 0.0
    g = P.run_gpu(p, n_ngb_tol=1.0)
    assert g["stats_density"]["n_unconverged"] == 0
    d = oracle.density_at(p.x, p.v, p.m, g["h"].astype(np.float64), p.box)
    assert np.all(np.abs(d["N"] - 48.0) <= 1.0 + 1e-4), float(np.abs(d["N"] - 48.0).max())
    orc = P.oracle_given_h(p, g["h"])
    P.compare(g, orc, np.arange(p.n))


@pytest.mark.parametrize("t", [0, 1])
def test_unquantised_positions_at_the_faces(t):
    """arbitrary fp32 positions (off the 2^-24 grid) crowded against every periodic face,
    including 0 and the largest fp32 below L; all particles compared, modes A and B."""
    p = workloads.edges_unquantised(t, n=4000)
    _modes(p)

def test_c5_full_size_sampled():
    """C5 (BASELINE configs[4]: 512^3 = 134,217,728 clustered particles, 512 clumps) on one
    B200 in one context: 2,000 seeded targets plus the 100 largest and 100 smallest h, modes A
    and B. The oracle runs on the particles within 2 h_max of a target (every source of their
    density and force sums, and of their neighbours' densities: the sums are exact), found by a
    grid hash of cell edge 2 h_max."""
    import torch

    import paper_1404_2303_b200 as sph
    p = workloads.c5()
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = sph.Context(sph.default_config(p.box, n_ngb_tol=1e-4, split_count=48, split_fraction=0.0))
    ctx.build_cells(t(p.x), None)
    d = ctx.density(t(p.v), t(p.m), t(p.u))
    f = ctx.force(t(p.v))
    g = {k: getattr(d, k).cpu().numpy() for k in ("h", "rho", "omega", "n_nbr", "div", "curl")}
    g.update({k: getattr(f, k).cpu().numpy() for k in ("a", "dudt", "vsig", "n_nbr_force")})
    assert d.stats["n_unconverged"] == 0
    ctx.close()
    del d, f
    torch.cuda.empty_cache()
    rng = np.random.default_rng(5)
    order = np.argsort(g["h"])
    T = np.unique(np.concatenate([rng.choice(p.n, 2000, replace=False), order[:100], order[-100:]]))
    # local particle set: every particle in the grid cells (edge 2 h_max) around a target's cell
    R = 2.0 * float(g["h"].max()) * 1.001
    nc = max(3, int(1.0 / R))
    cell = np.minimum((p.x * nc).astype(np.int64), nc - 1)
    cid = (cell[:, 0] * nc + cell[:, 1]) * nc + cell[:, 2]
    tc = cell[T]
    near = set()
    for ox in (-1, 0, 1):
        for oy in (-1, 0, 1):
            for oz in (-1, 0, 1):
                q = (tc + np.array([ox, oy, oz])) % nc
                near.update(((q[:, 0] * nc + q[:, 1]) * nc + q[:, 2]).tolist())
    sel = np.nonzero(np.isin(cid, np.fromiter(near, np.int64)))[0]
    del cell, cid
    loc = p.take(sel)
    tl = np.searchsorted(sel, T)
    h_or = oracle.solve_h(loc.x, loc.box, targets=tl)
    rel_h = np.abs(g["h"][T] - h_or) / h_or
    assert rel_h.max() <= P.TOL_H, float(rel_h.max())
    gl = {k: v[sel] for k, v in g.items()}
    orc = P.oracle_given_h(loc, gl["h"], targets=tl)
    P.compare(gl, orc, tl)
