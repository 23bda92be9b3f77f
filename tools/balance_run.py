"""Load balance of the slab partition on ONE GPU (NEXT-f3: work-weighted cuts).

The P ranks of a C5 slab decomposition are evaluated one after another on one GPU, each with
its own context over its owned particles and the halo it would receive (taken from the global
arrays; the exchange itself is not timed here), for two partitions:
  count  cuts at particle-count quantiles (the default),
  work   cuts at quantiles of slab.work_weights (n_nbr + n_nbr_force + WORK_FIXED) from the
         count run's outputs.
Per rank: owned / halo counts, build / density / force ms (CUDA events on the context's
stream, median of 3 after a warm-up). max / mean of the per-rank step time bounds the strong-
scaling efficiency of a P-GPU run from load balance alone: E <= T1 / (P x max_rank).

  python tools/balance_run.py [--n N] [--P 8] [--out profiles/round2/balance_c5.jsonl]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512 ** 3)
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--fixed", type=int, nargs="*", default=[])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_1404_2303_b200 as sph
    import workloads
    from paper_1404_2303_b200 import slab

    t0 = time.time()
    p = workloads.c5(n=args.n, n_clumps=max(8, int(512 * args.n / 512 ** 3)))
    print(f"generated {p.n} in {time.time() - t0:.0f} s", flush=True)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    tune = dict(split_count=48, split_fraction=0.0)
    Lx = p.box[0]
    out = []

    def emit(rec):
        out.append(rec)
        print(json.dumps(rec), flush=True)

    # T1 and the global h (the halo width each partition needs) from one context
    ctx = sph.Context(sph.default_config(p.box, **tune), stream=stream.cuda_stream)
    x = t(p.x)
    hist_n = ctx.x_histogram(x, 0.0, Lx, 8192).cpu().numpy()
    times = []
    for rep in range(3):
        ctx.build_cells(x, None)
        d = ctx.density(t(p.v), t(p.m), t(p.u))
        f = ctx.force(t(p.v))
        times.append(d.stats["ms_build"] + d.stats["ms_density"] + f.stats["ms_force"])
    T1 = float(np.median(times[1:]))
    h = d.h.cpu().numpy()
    nn = d.n_nbr.cpu().numpy().astype(np.int64)
    nf = f.n_nbr_force.cpu().numpy().astype(np.int64)
    F1 = int(f.stats["n_pairs"])
    del x, d, f
    ctx.close()
    torch.cuda.empty_cache()
    emit({"run": "single", "N": p.n, "T1_ms": T1, "F": F1})

    def need_width(edges):
        xs = p.x[:, 0].astype(np.float64)
        need = 0.0
        for e in edges[:-1] + [Lx]:
            dist = np.abs(xs - e)
            dist = np.minimum(dist, Lx - dist)
            near = dist < h
            if near.any():
                need = max(need, float(h[near].max()))
        return need * (1 + 1e-6)

    def face_need(e):
        """the halo width one cut needs: the largest h of a particle within h of it"""
        xs = p.x[:, 0].astype(np.float64)
        dist = np.abs(xs - e)
        dist = np.minimum(dist, Lx - dist)
        near = dist < h
        return float(h[near].max()) * (1 + 1e-6) if near.any() else 0.0

    T = 64   # face tiles per axis for the tile-width halo (tile edge >= the largest h near a face)

    def tile_width(e):
        """per face tile (y, z): the largest h of a particle within h of cut e in that tile,
        dilated over the 3 x 3 neighbouring tiles (a pair crosses at most one tile boundary
        when the tile edge is >= its reach)"""
        xs = p.x[:, 0].astype(np.float64)
        dist = np.abs(xs - e)
        dist = np.minimum(dist, Lx - dist)
        near = np.nonzero(dist < h)[0]
        ty = np.minimum((p.x[near, 1] / p.box[1] * T).astype(np.int64), T - 1)
        tz = np.minimum((p.x[near, 2] / p.box[2] * T).astype(np.int64), T - 1)
        W = np.zeros((T, T))
        np.maximum.at(W, (ty, tz), h[near])
        D = W.copy()
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                D = np.maximum(D, np.roll(np.roll(W, dy, 0), dz, 1))
        return D * (1 + 1e-6)

    def run_partition(name, edges, per_face=False, tiles=False):
        width = need_width(edges)
        fw = [face_need(e) for e in edges[:-1]] if per_face else [width] * args.P
        tw = [tile_width(e) for e in edges[:-1]] if tiles else None
        ranks = []
        for r in range(args.P):
            lo, hi = edges[r], edges[r + 1]
            w_lo, w_hi = (fw[r], fw[(r + 1) % args.P]) if per_face else (width, width)
            xs = p.x[:, 0]
            own = np.nonzero((xs >= lo) & (xs < hi))[0]
            dlo = (lo - xs) % Lx                      # distance below the lower face (periodic)
            dhi = (xs - hi) % Lx                      # distance above the upper face
            if tiles:
                ty = np.minimum((p.x[:, 1] / p.box[1] * T).astype(np.int64), T - 1)
                tz = np.minimum((p.x[:, 2] / p.box[2] * T).astype(np.int64), T - 1)
                wl, wh = tw[r][ty, tz], tw[(r + 1) % args.P][ty, tz]
                halo = np.nonzero(((dlo > 0) & (dlo <= wl)) | ((dhi >= 0) & (dhi < wh)))[0]
                w_lo, w_hi = float(tw[r].max()), float(tw[(r + 1) % args.P].max())
            else:
                halo = np.nonzero(((dlo > 0) & (dlo <= w_lo)) | ((dhi >= 0) & (dhi < w_hi)))[0]
            halo = np.setdiff1d(halo, own)
            idx = np.concatenate([own, halo])
            # the libsph check takes one width: the wider face's (the narrower face's halo is
            # complete for its own particles, which is what this timing needs)
            cfg = sph.default_config(p.box, **tune, rank=r, nranks=args.P, slab_lo=lo, slab_hi=hi,
                                     halo_width=max(w_lo, w_hi))
            c = sph.Context(cfg, stream=stream.cuda_stream)
            X, V, M, U = t(p.x[idx]), t(p.v[idx]), t(p.m[idx]), t(p.u[idx])
            ms = []
            for rep in range(4):
                c.build_cells_halo(X, own.size, None)
                d = c.density(V, M, U)
                f = c.force(X[: own.size])
                ms.append((d.stats["ms_build"], d.stats["ms_density"], f.stats["ms_force"]))
            ms = np.median(np.array(ms[1:]), axis=0)
            rec = {"run": name, "rank": r, "lo": lo, "hi": hi, "n_own": int(own.size), "n_halo": int(halo.size),
                   "width": width, "w_lo": w_lo, "w_hi": w_hi, "ms_build": float(ms[0]), "ms_density": float(ms[1]), "ms_force": float(ms[2]),
                   "ms_step": float(ms.sum()), "F": int(f.stats["n_pairs"]),
                   "sum_n_nbr": int(nn[own].sum()), "sum_n_nbr_force": int(nf[own].sum())}
            emit(rec)
            ranks.append(rec)
            del X, V, M, U, d, f
            c.close()
            torch.cuda.empty_cache()
        st = np.array([r["ms_step"] for r in ranks])
        emit({"run": name, "summary": True, "P": args.P, "max_ms": float(st.max()), "mean_ms": float(st.mean()),
              "imbalance": float(st.max() / st.mean()), "E_bound": T1 / (args.P * float(st.max())),
              "halo_over_owned": float(sum(r["n_halo"] for r in ranks) / p.n), "width": width})
        return ranks

    edges_n = slab.slab_cuts(hist_n, 0.0, Lx, args.P)
    run_partition("count", edges_n)
    run_partition("count, per-face width", edges_n, per_face=True)
    run_partition(f"count, {T}x{T} face-tile widths", edges_n, tiles=True)
    for fixed in args.fixed:
        w = (nn + nf + fixed).astype(np.float64)
        b = np.clip(np.floor(p.x[:, 0].astype(np.float64) / Lx * 8192).astype(np.int64), 0, 8191)
        hist_w = np.bincount(b, weights=w, minlength=8192)
        run_partition(f"work{fixed}", slab.slab_cuts(hist_w, 0.0, Lx, args.P))
    if args.out:
        with open(args.out, "w") as fh:
            for r in out:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
