"""How much would a better cold-start guess of h buy? C4 step time when the build starts from
h0 = converged h x exp(sigma N(0,1)) (a guess of log-spread sigma; the occupancy guess
k_guess_h has p10/p90 of guess/h 0.86/1.24, the cube-overlap estimate of
tools/guess_proto.py 0.87/1.13 after its bias), for a few list margins h_margin.
Also the cold start itself for reference.

  python tools/guess_quality_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1404_2303_b200 as sph
import workloads

p = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "C4")
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
base = dict(split_count=48, split_fraction=0.0)


def run(h0, **cfg):
    ctx = sph.Context(sph.default_config(p.box, **base, **cfg))
    res = []
    for _ in range(4):
        ctx.build_cells(x, h0)
        d = ctx.density(v, m, u)
        f = ctx.force(v)
        torch.cuda.synchronize()
        res.append((d.stats["ms_build"] + d.stats["ms_density"] + f.stats["ms_force"], d.stats["ms_kernel_walk_nb"],
                    d.stats["n_nb_entries"], d.stats["n_rebuilds"]))
    ctx.close()
    res.sort()
    return res[1], d.h.clone()


(cold, nbw, ent, reb), h = run(None)
print(json.dumps({"case": "cold (k_guess_h)", "ms_step": cold, "ms_walk_nb": nbw, "nb_entries": ent,
                  "rewalked": reb}), flush=True)
rng = np.random.default_rng(140423077)
z = rng.standard_normal(p.n).astype(np.float32)
for sigma in (0.0, 0.05, 0.1, 0.15, 0.25):
    h0 = (h * t(np.exp(sigma * z).astype(np.float32))).contiguous()
    for hm in (1.05, 1.1, 1.2, 1.3):
        (ms, nbw, ent, reb), _ = run(h0, h_margin=hm)
        print(json.dumps({"sigma": sigma, "h_margin": hm, "ms_step": ms, "ms_walk_nb": nbw, "nb_entries": ent,
                          "rewalked": reb}), flush=True)
