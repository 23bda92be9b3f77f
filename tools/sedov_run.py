"""Sedov blast (the paper's second test): an FCC lattice at rest with rho = 1
and a cold background, the energy E put into the particles near the centre, evolved with
the velocity-Verlet loop (integrate.Leapfrog). A point explosion in a uniform medium is
self-similar: the shock radius grows as R ~ (E t^2 / rho)^(1/5) (dimensional analysis,
exact), so log R against log t must have slope 2/5. R(t) = the radius of the peak of the
radially binned SPH density.
  python tools/sedov_run.py [cells_per_axis] [t_end]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph
from paper_1404_2303_b200.integrate import Leapfrog
from workloads.generators import quantise_positions


def setup(nc, E=1.0, p_amb=1e-6, g=5.0 / 3.0):
    base = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]])
    ijk = np.stack(np.meshgrid(*[np.arange(nc)] * 3, indexing="ij"), -1).reshape(-1, 1, 3)
    x64 = ((ijk + base[None] + 0.25) / nc).reshape(-1, 3)
    x = quantise_positions(x64, (1.0, 1.0, 1.0))
    n = x.shape[0]
    m = np.full(n, 1.0 / n, np.float32)
    u = np.full(n, p_amb / ((g - 1) * 1.0), np.float64)
    r = np.linalg.norm(x.astype(np.float64) - 0.5, axis=1)
    hot = r < 1.01 * np.sort(r)[30]          # the ~30 particles nearest the centre
    u[hot] += E / (m[0] * hot.sum())
    return x, np.zeros((n, 3), np.float32), m, u.astype(np.float32)


def shock_radius(x, rho, nbins=200):
    r = np.linalg.norm(x.astype(np.float64) - 0.5, axis=1)
    edges = np.linspace(0, 0.45, nbins + 1)
    idx = np.digitize(r, edges) - 1
    ok = (idx >= 0) & (idx < nbins)
    s = np.bincount(idx[ok], weights=rho[ok], minlength=nbins)
    c = np.bincount(idx[ok], minlength=nbins)
    prof = np.where(c > 0, s / np.maximum(c, 1), 0)
    k = int(np.argmax(prof))
    # the shock's leading edge: the outermost radius where the profile still exceeds the
    # midpoint between the background (1) and the peak (less noisy than the peak position)
    half = 0.5 * (1.0 + prof[k])
    above = np.nonzero(prof > half)[0]
    j = int(above.max())
    return 0.5 * (edges[j] + edges[j + 1]), float(prof[k])


def run(nc=32, t_end=0.05, n_snap=6):
    x, v, m, u = setup(nc)
    t = lambda q: torch.from_numpy(np.ascontiguousarray(q)).cuda()
    ctx = sph.Context(sph.default_config((1.0, 1.0, 1.0), n_ngb_tol=1e-3, split_count=48, split_fraction=0.0))
    lf = Leapfrog(ctx, t(x), t(v), t(m), t(u))
    E0 = lf.energy()
    snaps = np.geomspace(t_end / 8, t_end, n_snap)
    T, steps, out = 0.0, 0, []
    for ts in snaps:
        while T < ts - 1e-12:
            T += lf.step(min(lf.timestep(), ts - T))
            steps += 1
        R, peak = shock_radius(lf.x.cpu().numpy(), lf.rho.cpu().numpy().astype(np.float64))
        out.append((T, R, peak))
    ts_, rs_ = np.log([o[0] for o in out]), np.log([o[1] for o in out])
    slope = float(np.polyfit(ts_, rs_, 1)[0])
    res = {"n": int(x.shape[0]), "steps": steps, "snapshots": out, "slope": slope,
           "dE_over_E": (lf.energy() - E0) / abs(E0)}
    ctx.close()
    return res


if __name__ == "__main__":
    nc = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    te = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
    print(json.dumps(run(nc, te)))
