"""Binning + sort (a1-a3) throughput at a C5 shard size: the C5 recipe (clustered, cold h0)
at N particles on one GPU, the a1-a3 kernel time from sph_stats.ms_kernel_sort (CUDA events
around k_keys, the radix histogram and passes, k_pack and k_gather_vmu), the algorithmic bytes
of SURVEY 8(d): (28 + 24 x passes + 8 + 80) B per particle, against the measured HBM peak.
  python tools/binning_run.py [N=16777216] [reps=5]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1404_2303_b200 as sph
import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16777216
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = workloads.c5(n=n, n_clumps=max(8, int(512 * n / 512 ** 3)))
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
ms, passes, bits = [], 0, 0
for r in range(reps + 1):
    flush.zero_()
    ctx.build_cells(x, None)
    d = ctx.density(v, m, u)
    if r:
        ms.append(d.stats["ms_kernel_sort"])
    passes, bits = d.stats["sort_passes"], d.stats["sort_key_bits"]
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
bpp = 28 + 24 * passes + 8 + 80
t_ms = statistics.median(ms)
ach = n * bpp / (t_ms * 1e-3) / 1e9
print(json.dumps({"N": n, "workload": f"C5 recipe at N={n} ({p.meta['n_clumps']} clumps), cold h0", "sort_key_bits": bits,
                  "sort_passes": passes, "bytes_per_particle": bpp, "ms_a1_a3": t_ms, "ms_all": ms,
                  "achieved_GBs": ach, "peak_GBs": peaks["hbm_gbs"], "frac": ach / peaks["hbm_gbs"],
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs"}))
ctx.close()
