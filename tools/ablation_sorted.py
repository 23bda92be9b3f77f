"""the paper's sorted-interaction claim on the GPU path.

Runs one workload through the C ABI with leaves streamed whole through the box / sphere
filters (the bench path) and with every leaf presorted along the 13 directions and swept
through the windowed early exit of P:644-686 (sort_min_len = 0), for the count rule of the
bench and the paper's split rule (300 / 87.5 %). Results are the same in every
mode (the parity tests cover sort_min_len = 0); what changes is the number of sources the
walks stream and the time. Prints one JSON line per mode.
  python tools/ablation_sorted.py [C4|C2|C1] [reps]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1404_2303_b200 as sph
import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = workloads.make(name)
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
h0 = t(p.h0) if np.any(p.h0 > 0) else None
MODES = {
    "count48_streamed": dict(split_count=48, split_fraction=0.0, sort_min_len=64),
    "count48_presorted": dict(split_count=48, split_fraction=0.0, sort_min_len=0),
    "paper_streamed": dict(split_count=300, split_fraction=0.875, sort_min_len=1 << 30),
    "paper_presorted": dict(split_count=300, split_fraction=0.875, sort_min_len=0),
}
ref = None
for mode, kw in MODES.items():
    ctx = sph.Context(sph.default_config(p.box, flags=sph.SPH_F_SYNC | sph.SPH_F_COUNT_CANDIDATES, **kw))
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        ctx.build_cells(x, h0)
        d = ctx.density(v, m, u)
        f = ctx.force(v)
        torch.cuda.synchronize()
        sd, sf = d.stats, f.stats
        tot = sd["ms_build"] + sd["ms_density"] + sf["ms_force"]
        if best is None or tot < best[0]:
            best = (tot, sd, sf, d.h.clone())
    tot, sd, sf, h = best
    if ref is None:
        ref = h
    row = {"config": name, "mode": mode, "cfg": kw, "ms_step": tot, "ms_build": sd["ms_build"],
           "ms_density": sd["ms_density"], "ms_force": sf["ms_force"], "ms_walk_nb": sd["ms_kernel_walk_nb"],
           "ms_walk_union": sd["ms_kernel_walk_union"], "nb_sources": sd["n_nb_sources"],
           "union_sources": sd["n_union_sources"], "nb_entries": sd["n_nb_entries"],
           "union_entries": sd["n_pair_slots"], "F": sf["n_pairs"], "D": sd["n_directed"],
           "cells": sd["n_cells"], "leaves_or_groups": sd["n_leaves"],
           "h_max_rel_diff_vs_first_mode": float(((h - ref).abs() / ref).max())}
    row["nb_sources_per_entry"] = row["nb_sources"] / max(1, row["nb_entries"])
    print(json.dumps(row), flush=True)
    ctx.close()
