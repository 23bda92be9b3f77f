"""Dump the library's occupancy guess of h and the converged h for a config (GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
p = workloads.make(name)
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
x = t(p.x)
g = ctx.guess_h(x).cpu().numpy()
ctx.build_cells(x, None)
d = ctx.density(t(p.v), t(p.m), t(p.u))
np.save(f"gpurun_out/guess_{name}.npy", np.stack([g, d.h.cpu().numpy(), d.n_nbr.cpu().numpy().astype(np.float32)]))
r = g / d.h.cpu().numpy()
print("ratio guess/h: p1 %.3f p10 %.3f p50 %.3f p90 %.3f p99 %.3f p99.9 %.3f max %.3f" % tuple(np.percentile(r, [1, 10, 50, 90, 99, 99.9, 100])))
