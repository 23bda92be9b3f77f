"""Host-side pieces of bench.py's JSON line (no GPU): the ncu-derived tables it reads carry
every kernel its roofline objects name, and the issue-rate figure is instructions over time
against 148 SMs x 4 schedulers x 1 warp-instruction per clock at 1965 MHz."""
import json
import os

import bench

KERNELS = ("k_walk<MODE_NB>", "k_walk<MODE_FILL>", "k_force", "k_density")


def test_profile_tables_cover_the_roofline_kernels():
    for name in ("traffic.json", "issue.json"):
        d = json.load(open(os.path.join(bench.ROOT, "profiles", name)))
        for k in KERNELS:
            assert isinstance(d.get(k), int) and d[k] > 0, (name, k)


def test_issue_rate():
    assert abs(bench.ISSUE_PEAK_GINST - 1163.28) < 1e-9
    inst = json.load(open(os.path.join(bench.ROOT, "profiles", "issue.json")))["k_force"]
    r = bench.issue_from_profiles("k_force", 1.0)          # 1 ms launch
    assert r["warp_inst_per_launch"] == inst
    assert abs(r["achieved_ginst_s"] - inst / 1e6) < 1e-9
    assert abs(r["frac"] - inst / 1e6 / 1163.28) < 1e-12
    assert bench.issue_from_profiles("k_force", 0.0) is None
    assert bench.issue_from_profiles("no_such_kernel", 1.0) is None
    assert bench.traffic_from_profiles("no_such_kernel") is None


def test_reference_closure_reproduces_the_whole_evaluation():
    """The reference arm's per-target closure (h on the targets and every possible force
    partner, density and state of the partners, force on the targets) gives the same h, rho,
    a and du/dt as the oracle's whole-box evaluation, on a clustered input where partners by
    their own (larger) h occur."""
    import numpy as np

    import bench
    import oracle
    import workloads
    p = workloads.tiny(4, n=3000, clump_frac=0.5, n_dup=0)
    ref = oracle.evaluate_all(p.x, p.v, p.m, p.u, p.box)
    bench.oracle_closure_setup(p)
    assert np.all(bench._G["hb"] >= ref["h"])                 # the bound holds
    T = np.sort(np.random.default_rng(3).choice(p.n, 60, replace=False))
    bench._G["keep"] = True
    work, _ = bench._w_closure(T)
    k = bench._G.pop("kept")
    bench._G.pop("keep")
    assert work > 0
    assert np.allclose(k["h"], ref["h"][T], rtol=1e-12)
    assert np.allclose(k["rho"], ref["rho"][T], rtol=1e-12)
    scale = np.abs(ref["a"]).max()
    assert np.abs(k["a"] - ref["a"][T]).max() <= 1e-10 * scale
    assert np.abs(k["dudt"] - ref["dudt"][T]).max() <= 1e-10 * np.abs(ref["dudt"]).max()
