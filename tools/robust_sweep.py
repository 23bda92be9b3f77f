"""Adversarial configuration sweep: each case through the C ABI, then the oracle's N(h) at
the GPU's h and its own root for a sample (+ the extreme h) -> max |N - 48|, max h error."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads, oracle

def case(name, p, h0=None, **cfg):
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    kw = dict(split_count=48, split_fraction=0.0, n_ngb_tol=1e-4); kw.update(cfg)
    ctx = sph.Context(sph.default_config(p.box, **kw))
    ctx.build_cells(t(p.x), None if h0 is None else t(h0))
    d = ctx.density(t(p.v), t(p.m), t(p.u), check=False)
    f = ctx.force(t(p.v))
    h = d.h.cpu().numpy()
    rng = np.random.default_rng(0)
    o = np.argsort(h)
    s = np.unique(np.concatenate([o[:100], o[-100:], rng.choice(p.n, min(p.n, 1500), replace=False)]))
    den = oracle.density_at(p.x, p.v, p.m, h, p.box, targets=s)
    hr = oracle.solve_h(p.x, p.box, targets=s)
    out = {"case": name, "n": p.n, "unconv": d.stats["n_unconverged"], "N_err_max": float(np.abs(den["N"] - 48).max()),
           "h_rel_max": float(np.abs(h[s] / hr - 1).max()), "a_finite": bool(np.isfinite(f.a.cpu().numpy()).all())}
    ctx.close()
    print(json.dumps(out), flush=True)

c1, c2, c3, c4 = workloads.c1(), workloads.c2(), workloads.c3(), workloads.c4()
case("C1", c1)
case("C2", c2, h0=c2.h0)
case("C3", c3, h0=c3.h0)
case("C4", c4)
case("C4 paper rule", c4, split_count=300, split_fraction=0.875)
case("C4 presort", c4, sort_min_len=0)
rng = np.random.default_rng(7)
# warm starts from a converged h with large errors
ctx = sph.Context(sph.default_config(c4.box, split_count=48, split_fraction=0.0))
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ctx.build_cells(t(c4.x)); hc = ctx.density(t(c4.v), t(c4.m), t(c4.u)).h.cpu().numpy(); ctx.close()
for e in [0.05, 0.3, 0.6]:
    case(f"C4 warm +-{e}", c4, h0=(hc * (1 + e * rng.uniform(-1, 1, c4.n))).astype(np.float32))
case("C4 warm all 3x too small", c4, h0=(hc / 3).astype(np.float32))
case("C4 warm all 3x too large", c4, h0=np.minimum(hc * 3, 0.3).astype(np.float32))
for sd in range(3):
    p = workloads.tiny(20 + sd, n=8000, clump_frac=0.5, n_dup=3)
    p.h0[:] = 0
    case(f"tiny{sd}", p)
case("C1 tol 1 (paper)", c1, n_ngb_tol=1.0)
