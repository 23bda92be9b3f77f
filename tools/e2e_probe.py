import os, sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads
p = workloads.c4(); N = p.n
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hx, hv, hm, hu = pin(p.x), pin(p.v), pin(p.m), pin(p.u)
hod = dict(h=torch.empty(N).pin_memory(), rho=torch.empty(N).pin_memory())
hof = dict(a=torch.empty(N, 3).pin_memory(), dudt=torch.empty(N).pin_memory())
dev = torch.device("cuda:0")
dx, dv, dm, du = (t.to(dev) for t in (hx, hv, hm, hu))
dod = dict(h=torch.empty(N, device=dev), rho=torch.empty(N, device=dev))
dof = dict(a=torch.empty(N, 3, device=dev), dudt=torch.empty(N, device=dev))
for label, X, V, M, U, od, of in (("device", dx, dv, dm, du, dod, dof), ("host", hx, hv, hm, hu, hod, hof)):
    for rep in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx.build_cells(X, None); t1 = time.perf_counter()
        d = ctx.density(V, M, U, out=od); t2 = time.perf_counter()
        f = ctx.force(V, out=of); t3 = time.perf_counter()
        print(label, "wall build %.2f density %.2f force %.2f ms" % (1e3*(t1-t0), 1e3*(t2-t1), 1e3*(t3-t2)),
          "events build %.2f density %.2f force %.2f" % (d.stats["ms_build"], d.stats["ms_density"], f.stats["ms_force"]))
