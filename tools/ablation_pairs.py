"""the paper's cell-pair density loops, naive vs presorted sweeps
with early exit, on a uniform grid of edge >= max h, against the hot path's density
(rho at 1e-5) and with the window-pass / in-range rates per neighbour class (R9: the paper's
33.5 / 16.2 / 3.6 % for face / edge / corner neighbours of cells of edge h).
  python tools/ablation_pairs.py [C1 C2 C2-exact C4 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1404_2303_b200 as sph
import workloads

names = sys.argv[1:] or ["C2-exact", "C1", "C2", "C4"]
dev = torch.device("cuda:0")
for name in names:
    p = workloads.make(name)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
    ctx.build_cells(t(p.x), t(p.h0) if np.any(p.h0 > 0) else None)
    d = ctx.density(t(p.v), t(p.m), t(p.u))
    rho = d.rho.clone()
    row = {"workload": name, "N": p.n}
    for mode in ("naive", "sorted"):
        best = None
        for rep in range(3):
            out = torch.empty_like(rho)
            c = ctx.pair_ablation(mode == "sorted", out)
            if best is None or c["ns_loop"] < best["ns_loop"]:
                best = c
        rel = float(((out - rho).abs() / rho).max())
        pf, pe, pc = best["pairs_face"], best["pairs_edge"], best["pairs_corner"]
        row[mode] = {"ms_loop": best["ns_loop"] / 1e6, "ms_presort": best["ns_presort"] / 1e6, "tests": best["tests"],
                     "hits": best["hits"], "cells_x": best["cells_x"], "rho_rel_max_vs_hot_path": rel,
                     "window_pass_rate": {"face": best["pass_face"] / max(pf, 1), "edge": best["pass_edge"] / max(pe, 1),
                                          "corner": best["pass_corner"] / max(pc, 1)},
                     "in_range_rate": {"face": best["inrange_face"] / max(pf, 1), "edge": best["inrange_edge"] / max(pe, 1),
                                       "corner": best["inrange_corner"] / max(pc, 1)}}
    row["naive_over_sorted_loop_time"] = row["naive"]["ms_loop"] / row["sorted"]["ms_loop"]
    row["naive_over_sorted_tests"] = row["naive"]["tests"] / row["sorted"]["tests"]
    print(json.dumps(row), flush=True)
    ctx.close()
