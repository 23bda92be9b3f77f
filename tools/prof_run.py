"""Warm timing / profiling driver: one config through the C ABI `reps` times (device
arrays, cold h0 as the config specifies); prints the per-call stats of the last rep.
  python tools/prof_run.py C4 [reps] [json cfg overrides]
Under ncu, capture the last rep with --launch-skip / -k filters."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1404_2303_b200 as sph
import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kw = dict(split_count=48, split_fraction=0.0)
if len(sys.argv) > 3:
    kw.update(json.loads(sys.argv[3]))
p = workloads.make(name)
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
h0 = t(p.h0) if np.any(p.h0 > 0) else None
ctx = sph.Context(sph.default_config(p.box, **kw))
for r in range(reps):
    if r == reps - 1:
        os.environ["SPH_DEBUG"] = os.environ.get("SPH_DEBUG_LAST", "0")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.build_cells(x, h0)
    d = ctx.density(v, m, u)
    f = ctx.force(v)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
sd, sf = d.stats, f.stats
F = sf["n_pairs"]
tot = sd["ms_build"] + sd["ms_density"] + sf["ms_force"]
print(json.dumps({"config": name, "cfg": kw, "wall_ms": wall * 1e3, "ms_build": sd["ms_build"],
                  "ms_density": sd["ms_density"], "ms_force": sf["ms_force"], "ms_total_events": tot,
                  "ms_kernel_density_full": sd["ms_kernel_density_full"], "ms_kernel_force": sf["ms_kernel_force"],
                  "F": F, "D": sd["n_directed"], "rate": 2 * F / (tot * 1e-3), "h_iters": sd["h_iters"],
                  "groups": sd["n_leaves"], "cells": sd["n_cells"], "levels": sd["n_levels"],
                  "list_dens": sd["n_pair_slots"], "list_rebuild_groups": sd["n_rebuilds"],
                  "cand_dens_first": sd["n_candidates"], "cand_force": sf["n_candidates"]}))
ctx.close()
