"""Dump one evaluation's outputs (h, rho, a, du/dt, counts) of the library in SPH_LIB, for
bitwise A/B comparisons of kernel variants:
  SPH_LIB=... python tools/ab_outputs.py out.npz [config]
  python tools/ab_outputs.py --cmp a.npz b.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        x, y = a[k].astype(np.float64), b[k].astype(np.float64)
        print(k, "equal" if np.array_equal(a[k], b[k]) else
              f"differ: max |d| {np.abs(x - y).max():.3g}, max rel {np.abs(x - y).max() / max(np.abs(x).max(), 1e-30):.3g}")
    sys.exit(0)
import torch
import paper_1404_2303_b200 as sph
import workloads
p = workloads.make(sys.argv[2] if len(sys.argv) > 2 else "C4")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
h0 = t(p.h0) if np.any(p.h0 > 0) else None
ctx.build_cells(x, h0)
d = ctx.density(v, m, u)
f = ctx.force(v)
np.savez(sys.argv[1], h=d.h.cpu().numpy(), rho=d.rho.cpu().numpy(), n=d.n_nbr.cpu().numpy(), a=f.a.cpu().numpy(),
         dudt=f.dudt.cpu().numpy(), nf=f.n_nbr_force.cpu().numpy())
print("F", f.stats["n_pairs"], "ms", d.stats["ms_build"], d.stats["ms_density"], f.stats["ms_force"])
