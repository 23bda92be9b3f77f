"""Edge cases and degenerate inputs through the C ABI (SURVEY 8(b) error conventions,
8(c) O4 uniqueness of the h root):

  * ragged small N (a few warps, h near the L/2 cap, every particle sees wrapped images),
    full parity against the oracle;
  * too few particles for N_ngb = 48 below h = L/2: SPH_E_NOCONV, outputs still written
    and finite (the §8(b) NOCONV contract);
  * more than 4 coincident particles: N(h) >= (32/3) k > 48 for every h > 0, so no root
    exists (O4); those particles stop at the h floor and are reported unconverged, their
    neighbours converge, no output is inf or NaN;
  * N = 0: SPH_E_ARG.
"""
import numpy as np
import pytest

import oracle
from workloads.generators import Particles, quantise_positions

from . import parity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests must run on the B200 box")
    from paper_1404_2303_b200 import build
    build.build()


def _uniform(n, seed, extra=None):
    rng = np.random.default_rng(seed)
    x64 = rng.random((n, 3))
    if extra is not None:
        x64 = np.concatenate([x64, extra])
    n = x64.shape[0]
    x = quantise_positions(x64, (1.0, 1.0, 1.0))
    v = (0.1 * rng.standard_normal((n, 3))).astype(np.float32)
    m = rng.uniform(0.5, 1.5, n).astype(np.float32) / n
    u = rng.uniform(0.5, 2.0, n).astype(np.float32)
    return Particles("edge", (1.0, 1.0, 1.0), x, v, m, u, np.zeros(n, np.float32))


def _run(p, check=True):
    import torch

    import paper_1404_2303_b200 as sph
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = sph.Context(sph.default_config(p.box, n_ngb_tol=1e-4))
    ctx.build_cells(t(p.x))
    d = ctx.density(t(p.v), t(p.m), t(p.u), check=check)
    f = ctx.force(t(p.v))
    out = {k: getattr(d, k).cpu().numpy() for k in ("h", "rho", "omega", "div", "curl")}
    out.update({k: getattr(f, k).cpu().numpy() for k in ("a", "dudt", "vsig")})
    out["stats_density"] = d.stats
    ctx.close()
    return out


@pytest.mark.parametrize("n", [200, 255, 257])
def test_ragged_small_n_full_parity(n):
    """A handful of warps, ragged last group, h up to ~0.47 L (wrapped images everywhere)."""
    p = _uniform(n, 100 + n)
    g = P.run_gpu(p)
    h_or = oracle.solve_h(p.x, p.box)
    assert np.abs(g["h"] / h_or - 1).max() <= P.TOL_H
    rep = P.compare(g, P.oracle_given_h(p, g["h"]), np.arange(n))
    assert g["stats_density"]["n_unconverged"] == 0, rep


@pytest.mark.parametrize("n", [1, 5, 40])
def test_too_few_particles_noconv(n):
    import paper_1404_2303_b200 as sph
    p = _uniform(n, 7 + n)
    with pytest.raises(sph.SphError) as e:
        _run(p)
    assert e.value.status == sph.SPH_E_NOCONV
    g = _run(p, check=False)
    assert g["stats_density"]["n_unconverged"] == n
    for k in ("h", "rho", "a", "dudt"):
        assert np.all(np.isfinite(g[k])), k
    assert np.all(g["h"] < 0.5)                       # h stays below the L/2 cap


def test_coincident_cluster_has_no_root():
    import paper_1404_2303_b200 as sph
    k = 60
    p = _uniform(400, 3, extra=np.full((k, 3), 0.3125))
    with pytest.raises(sph.SphError) as e:
        _run(p)
    assert e.value.status == sph.SPH_E_NOCONV
    g = _run(p, check=False)
    for key in ("h", "rho", "omega", "a", "dudt", "vsig"):
        assert np.all(np.isfinite(g[key])), key
    assert g["stats_density"]["n_unconverged"] == k
    cl = np.arange(400, 400 + k)
    assert np.all(g["h"][cl] < 1e-5)                  # stopped at the floor
    # every other particle converged to the oracle's root (the cluster counts k times)
    bg = np.arange(400)
    h_or = oracle.solve_h(p.x, p.box, targets=bg)
    assert np.abs(g["h"][bg] / h_or - 1).max() <= P.TOL_H


def test_empty_input():
    import torch

    import paper_1404_2303_b200 as sph
    ctx = sph.Context(sph.default_config((1.0, 1.0, 1.0)))
    with pytest.raises(sph.SphError) as e:
        ctx.build_cells(torch.zeros(0, 3, device="cuda"))
    assert e.value.status == sph.SPH_E_ARG
    ctx.close()
