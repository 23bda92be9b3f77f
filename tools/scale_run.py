"""Single-GPU capacity / timing run of the C5 recipe (512 clumps, clustered) at a given N,
with optional sampled parity against the oracle.
  python tools/scale_run.py N [n_parity_samples]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1404_2303_b200 as sph
import workloads

n = int(sys.argv[1])
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t0 = time.time()
p = workloads.c5(n=n, n_clumps=max(8, int(512 * n / 512 ** 3)))
tgen = time.time() - t0
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
res = []
for rep in range(2):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ctx.build_cells(x, None)
    d = ctx.density(v, m, u)
    f = ctx.force(v)
    torch.cuda.synchronize()
    sd, sf = d.stats, f.stats
    res.append({"wall_ms": 1e3 * (time.perf_counter() - w0), "ms_build": sd["ms_build"], "ms_density": sd["ms_density"],
                "ms_force": sf["ms_force"], "F": sf["n_pairs"], "groups": sd["n_leaves"], "walk_nb": sd["ms_kernel_walk_nb"],
                "hsolve": sd["ms_kernel_hsolve"], "walk_union": sd["ms_kernel_walk_union"],
                "k_density": sd["ms_kernel_density_full"], "k_force": sf["ms_kernel_force"]})
free, total = torch.cuda.mem_get_info()
last = res[-1]
tot = last["ms_build"] + last["ms_density"] + last["ms_force"]
print(json.dumps({"N": n, "gen_s": round(tgen, 1), "ms_step": tot, "rate": 2 * last["F"] / (tot * 1e-3),
                  "mem_used_GB": round((total - free) / 1e9, 1), **last}))
if ns:
    import oracle
    from tests import parity as P
    g = {"h": d.h.cpu().numpy(), "rho": d.rho.cpu().numpy(), "omega": d.omega.cpu().numpy(),
         "n_nbr": d.n_nbr.cpu().numpy(), "div": d.div.cpu().numpy(), "curl": d.curl.cpu().numpy(),
         "a": f.a.cpu().numpy(), "dudt": f.dudt.cpu().numpy(), "vsig": f.vsig.cpu().numpy(),
         "n_nbr_force": f.n_nbr_force.cpu().numpy()}
    rng = np.random.default_rng(5)
    tt = np.sort(rng.choice(n, ns, replace=False))
    h_or = oracle.solve_h(p.x, p.box, targets=tt)
    rel = np.abs(g["h"][tt] - h_or) / h_or
    orc = P.oracle_given_h(p, g["h"], targets=tt)
    rep = P.compare(g, orc, tt)
    print(json.dumps({"parity_samples": ns, "h_rel_max": float(rel.max()), **rep}))
ctx.close()
