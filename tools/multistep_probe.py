"""Sod with individual time steps (integrate.MultiStep) vs the global step (Leapfrog)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import numpy as np, torch
import paper_1404_2303_b200 as sph
from paper_1404_2303_b200.integrate import MultiStep
import sod_run
from tests import sod_exact as S


def run(nl=40, t_end=0.1, n_bins=4):
    x, v, m, u, rho_r = sod_run.setup(nl)
    t = lambda q: torch.from_numpy(np.ascontiguousarray(q)).cuda()
    ctx = sph.Context(sph.default_config((2.0, 1.0, 1.0), n_ngb_tol=1e-3, split_count=48, split_fraction=0.0))
    ms = MultiStep(ctx, t(x), t(v), t(m), t(u), dt_max=t_end / 4, n_bins=n_bins)
    E0 = ms.synced_energy()
    steps = 0
    while ms.time() < t_end - 1e-12:
        ms.step(); steps += 1
    E1 = ms.synced_energy()
    xs = ms.x.cpu().numpy().astype(np.float64); rho = ms.rho.cpu().numpy().astype(np.float64)
    px = xs[:, 0]
    sel1 = np.abs(px - 1.0) < 0.4
    ex1 = S.density((px[sel1] - 1.0) / t_end, 4.0, 0.0, 1.0, rho_r, 0.0, 0.1795)
    l1 = float(np.abs(rho[sel1] - ex1).sum() / np.abs(ex1).sum())
    bins = torch.bincount(torch.log2(ms.step_ticks.float()).long(), minlength=n_bins + 1).tolist()
    out = {"n": int(xs.shape[0]), "substeps": steps, "evaluations_over_n": ms.evaluations / xs.shape[0],
           "L1_rho": l1, "dE_over_E": (E1 - E0) / abs(E0), "bins_at_end": bins}
    ctx.close()
    return out


if __name__ == "__main__":
    print(json.dumps(run(int(sys.argv[1]) if len(sys.argv) > 1 else 40)))
