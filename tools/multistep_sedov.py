"""Sedov blast with individual time steps (integrate.MultiStep + limiter) vs the global
step: shock radius, energy, and how many particle evaluations each needed."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import numpy as np, torch
import paper_1404_2303_b200 as sph
from paper_1404_2303_b200.integrate import MultiStep
import sedov_run


def run(nc=32, t_end=0.05, n_bins=8, limiter=True):
    x, v, m, u = sedov_run.setup(nc)
    t = lambda q: torch.from_numpy(np.ascontiguousarray(q)).cuda()
    ctx = sph.Context(sph.default_config((1.0, 1.0, 1.0), n_ngb_tol=1e-3, split_count=48, split_fraction=0.0))
    ms = MultiStep(ctx, t(x), t(v), t(m), t(u), dt_max=t_end / 2, n_bins=n_bins, limiter=limiter)
    E0 = ms.synced_energy()
    steps = 0
    while ms.time() < t_end - 1e-12:
        ms.step(); steps += 1
    E1 = ms.synced_energy()
    R, peak = sedov_run.shock_radius(ms.x.cpu().numpy(), ms.rho.cpu().numpy().astype(np.float64))
    out = {"n": int(x.shape[0]), "substeps": steps, "evaluations_over_n": ms.evaluations / x.shape[0],
           "R": R, "R_over_sedov": R / (1.152 * (t_end ** 2) ** 0.2), "peak": peak, "dE_over_E": (E1 - E0) / abs(E0),
           "bins": torch.bincount(torch.log2(ms.step_ticks.float()).long()).tolist()}
    ctx.close()
    return out


if __name__ == "__main__":
    print(json.dumps(run(limiter=("--no-limiter" not in sys.argv))))
