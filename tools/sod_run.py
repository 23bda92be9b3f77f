"""The paper's Sod-shock test (rho 4 / 1, P 1 / 0.1795) in a 2x1x1 periodic box
of two cubic lattices, evolved with the velocity-Verlet loop (integrate.Leapfrog) and
compared with the exact Riemann solution at both interfaces (tests/sod_exact.py).
  python tools/sod_run.py [n_left_per_axis] [t_end]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph
from paper_1404_2303_b200.integrate import Leapfrog
from tests import sod_exact as S
from workloads.generators import quantise_positions


def setup(nl):
    g = 5.0 / 3.0
    nr = int(round(nl * 4 ** (-1 / 3)))
    ax = (np.arange(nl) + 0.5) / nl
    L = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    ar = (np.arange(nr) + 0.5) / nr
    R = np.stack(np.meshgrid(ar, ar, ar, indexing="ij"), -1).reshape(-1, 3)
    R[:, 0] += 1.0
    x = quantise_positions(np.concatenate([L, R]), (2.0, 1.0, 1.0))
    m0 = 4.0 / nl ** 3
    rho_r = m0 * nr ** 3
    n = x.shape[0]
    m = np.full(n, m0, np.float32)
    P = np.concatenate([np.full(nl ** 3, 1.0), np.full(nr ** 3, 0.1795)])
    rho = np.concatenate([np.full(nl ** 3, 4.0), np.full(nr ** 3, rho_r)])
    u = (P / ((g - 1) * rho)).astype(np.float32)
    return x, np.zeros((n, 3), np.float32), m, u, rho_r


def run(nl=40, t_end=0.1):
    x, v, m, u, rho_r = setup(nl)
    t = lambda q: torch.from_numpy(np.ascontiguousarray(q)).cuda()
    ctx = sph.Context(sph.default_config((2.0, 1.0, 1.0), n_ngb_tol=1e-3, split_count=48, split_fraction=0.0))
    lf = Leapfrog(ctx, t(x), t(v), t(m), t(u))
    E0, P0 = lf.energy(), lf.momentum()
    T, steps = 0.0, 0
    while T < t_end:
        T += lf.step(min(lf.timestep(), t_end - T))
        steps += 1
    xs = lf.x.cpu().numpy().astype(np.float64)
    rho = lf.rho.cpu().numpy().astype(np.float64)
    px = xs[:, 0]
    # interface at x = 1 (dense left) and at x = 0 = 2 (dense right, mirrored)
    sel1 = np.abs(px - 1.0) < 0.4
    ex1 = S.density((px[sel1] - 1.0) / T, 4.0, 0.0, 1.0, rho_r, 0.0, 0.1795)
    d0 = np.where(px > 1.0, px - 2.0, px)
    sel0 = np.abs(d0) < 0.4
    ex0 = S.density(d0[sel0] / T, rho_r, 0.0, 0.1795, 4.0, 0.0, 1.0)
    l1 = lambda a, b: float(np.abs(a - b).sum() / np.abs(b).sum())
    res = {"n": int(xs.shape[0]), "steps": steps, "t": T, "L1_rho_interface_1": l1(rho[sel1], ex1),
           "L1_rho_interface_0": l1(rho[sel0], ex0), "dE_over_E": (lf.energy() - E0) / abs(E0),
           "dP_max": float((lf.momentum() - P0).abs().max())}
    ctx.close()
    return res


if __name__ == "__main__":
    nl = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    te = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
    print(json.dumps(run(nl, te)))
