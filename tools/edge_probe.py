"""Probe edge cases through the C ABI (prints status / stats)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph
dev = torch.device("cuda:0")
def run(name, x, m=None):
    n = x.shape[0]
    ctx = sph.Context(sph.default_config((1.0, 1.0, 1.0), n_ngb_tol=1e-4))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)
    try:
        ctx.build_cells(t(x))
        d = ctx.density(t(np.zeros((n, 3))), t(np.full(n, 1.0 / n) if m is None else m), t(np.ones(n)), check=False)
        print(name, "n", n, "stats unconv", d.stats["n_unconverged"], "h range", float(d.h.min()), float(d.h.max()), "rho", float(d.rho.min()))
        f = ctx.force(t(np.zeros((n, 3))))
        print("   force ok, |a|max", float(f.a.abs().max()))
    except sph.SphError as e:
        print(name, "n", n, "-> SphError", e.status, str(e)[:150])
    ctx.close()
rng = np.random.default_rng(1)
for n in [1, 5, 40, 90, 97, 128, 200, 31, 32, 33]:
    run(f"uniform", rng.random((n, 3)))
run("coincident100", np.full((100, 3), 0.3))
run("two_clusters", np.concatenate([np.full((60, 3), 0.3), rng.random((200, 3))]))
try:
    ctx = sph.Context(sph.default_config((1.0, 1.0, 1.0)))
    ctx.build_cells(torch.zeros(0, 3, device=dev))
    print("n=0 accepted")
except sph.SphError as e:
    print("n=0 -> SphError", e.status, str(e)[:100])
