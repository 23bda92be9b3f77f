"""Quick GPU debug run: one config through the C ABI, stats + parity summary."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads, oracle
from tests import parity as P

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
p = workloads.make(name) if not name.startswith("tiny") else workloads.tiny(int(name[4:]), n=4000, clump_frac=0.3, n_dup=5)
if name.startswith("tiny"): p.h0[:] = 0
t0 = time.time()
import json
cfgkw = json.loads(os.environ.get("SPH_DBG_CFG", "{}"))
g = P.run_gpu(p, **cfgkw)
print(name, "gpu wall", time.time() - t0, flush=True)
print("density stats", g["stats_density"])
print("force stats", g["stats_force"])
print("h range", g["h"].min(), g["h"].max(), "nan?", np.isnan(g["rho"]).sum(), np.isnan(g["a"]).sum())
rng = np.random.default_rng(0)
t = np.sort(rng.choice(p.n, min(ns, p.n), replace=False))
t1 = time.time()
h_or = oracle.solve_h(p.x, p.box, targets=t)
print("mode A h rel max", np.max(np.abs(g["h"][t] - h_or) / h_or), "oracle", time.time() - t1, flush=True)
orc = P.oracle_given_h(p, g["h"], targets=t)
try:
    print("mode B", P.compare(g, orc, t))
except AssertionError as e:
    print("PARITY FAIL", e)
    dn = g["n_nbr"][t] - orc["n_nbr"]
    print("n_nbr diff hist", np.unique(dn, return_counts=True))
    rr = np.abs(g["rho"][t] - orc["rho"]) / orc["rho"]
    print("rho rel worst", np.sort(rr)[-5:])
    ea = np.linalg.norm(g["a"][t] - orc["a"], axis=1) / orc["S_a"]
    print("a worst", np.sort(ea)[-5:])
bad = np.argsort(-np.abs(g["h"][t] - h_or) / h_or)[:5]
print("worst h:", [(int(t[b]), float(g["h"][t[b]]), float(h_or[b])) for b in bad])
