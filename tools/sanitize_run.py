"""One evaluation (build + density + force) of C1 and of a tiny clumped case with
duplicates, for compute-sanitizer (memcheck / racecheck / synccheck), plus the code paths the
default configuration does not reach: the paper's split rule with every leaf presorted (the
13-direction sweeps), the neighbour-row overflow pool, and the interaction-list slab overflow.
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1404_2303_b200 as sph
import workloads

CASES = [
    ("C1 bench config", workloads.c1, dict(split_count=48, split_fraction=0.0)),
    ("tiny clumped + dups", lambda: workloads.tiny(4, n=3000, clump_frac=0.4, n_dup=5), {}),
    ("tiny presort every leaf", lambda: workloads.tiny(5, n=3000, clump_frac=0.4, n_dup=3),
     dict(split_count=300, split_fraction=0.875, sort_min_len=0)),
    ("tiny row overflow + pool", lambda: workloads.tiny(6, n=3000, clump_frac=0.4, n_dup=2),
     dict(split_count=48, split_fraction=0.0, row_cap=64)),
    ("C1 list slab overflow", workloads.c1, dict(split_count=48, split_fraction=0.0, list_cap=64)),
]

dev = torch.device("cuda:0")
for name, make, cfg in CASES:
    p = make()
    if name.startswith("tiny"):
        p.h0[:] = 0.0
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = sph.Context(sph.default_config(p.box, flags=sph.SPH_F_SYNC | sph.SPH_F_DIAGNOSTICS, **cfg))
    ctx.build_cells(t(p.x))
    d = ctx.density(t(p.v), t(p.m), t(p.u))
    f = ctx.force(t(p.v))
    torch.cuda.synchronize()
    print(f"{name}: n={p.n} F={f.stats['n_pairs']} D={d.stats['n_directed']} launches={ctx.kernel_launches}",
          flush=True)
    ctx.close()
print("sanitize_run done")
