"""Where the e2e time goes: sph_step on C4 with device arrays vs pinned host arrays
(per-call CUDA-event phases and wall time; 5 reps each, last 3 printed)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads
p = workloads.c4(); N = p.n
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hx, hv, hm, hu = pin(p.x), pin(p.v), pin(p.m), pin(p.u)
dev = torch.device("cuda:0")
dx, dv, dm, du = (t.to(dev) for t in (hx, hv, hm, hu))
ho = dict(h=torch.empty(N).pin_memory(), rho=torch.empty(N).pin_memory(), a=torch.empty(N, 3).pin_memory(),
          dudt=torch.empty(N).pin_memory())
do = {k: torch.empty_like(v, device=dev) for k, v in ho.items()}
for label, ins, out in (("device", (dx, dv, dm, du), do), ("host", (hx, hv, hm, hu), ho),
                        ("x-host", (hx, dv, dm, du), ho), ("vmu-host", (dx, hv, hm, hu), ho)):
    for rep in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d, f = ctx.step(*ins, out=out)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        if rep >= 2:
            sd, sf = d.stats, f.stats
            print(f"{label:8s} wall {1e3*(t1-t0):.3f} ms  build {sd['ms_build']:.3f} density {sd['ms_density']:.3f} "
                  f"force {sf['ms_force']:.3f} (kernels: walk_nb {sd['ms_kernel_walk_nb']:.3f} union "
                  f"{sd['ms_kernel_walk_union']:.3f} dens {sd['ms_kernel_density_full']:.3f} force {sf['ms_kernel_force']:.3f})")
