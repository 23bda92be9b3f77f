import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads, oracle
p = workloads.make("C4")
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0, n_ngb_tol=1e-4))
ctx.build_cells(t(p.x), None)
d = ctx.density(t(p.v), t(p.m), t(p.u), check=False)
print("unconv", d.stats["n_unconverged"], "h_iters", d.stats["h_iters"])
h = d.h.cpu().numpy()
# find particles whose N(h) is off: oracle N at the GPU h for a sample of particles with extreme h
idx = np.argsort(h)
sample = np.unique(np.concatenate([idx[:200], idx[-200:], np.random.default_rng(0).choice(p.n, 3000, replace=False)]))
den = oracle.density_at(p.x, p.v, p.m, h, p.box, targets=sample)
N = den["N"]
bad = np.abs(N - 48) > 1e-3
print("sampled", sample.size, "bad", bad.sum())
for i in np.nonzero(bad)[0][:10]:
    print(int(sample[i]), "h", h[sample[i]], "N", N[i], "n_nbr", int(den["n_nbr"][i]))
