// lists.cuh — interaction lists (neighbour finding, section 3.2-3.3).
//
// The paper finds the interacting pairs through cell pairs: every particle sits in a cell
// whose edge is at least its h, so its partners lie in the 26 neighbouring cells
// (P:471-499); pairs of large cells are refined into pairs of their children;
// and the particles of the two cells of a pair are swept in the order of their projection
// onto the axis joining the cells, so the sweep stops at the first particle whose projected
// distance exceeds h (P:644-698, 13 presorted directions per cell).
//
// On the GPU the same search is done ONCE per structure, per target group (<= 32
// consecutive particles of one leaf, one warp), and its result -- the group's candidate
// sources -- is stored as a flat list that every density pass (the h iteration) and the
// force pass stream through (the paper reuses its sorts for both loops):
//   1. the cells within reach of the group: the top cells around the group's bounding box
//      (with their periodic images), refined recursively into their children
//      while the child's box is within reach (the pair refinement of P:523-532, decided
//      per child box instead of per cell pair);
//   2. in a reached leaf, the sources are swept in the leaf's presorted order along the
//      canonical direction joining the group and the leaf, stopping at the first source
//      whose projection lies beyond the window (the sorted sweep of P:644-669, R6, R20);
//      leaves without a sorted list are swept whole;
//   3. every swept source is kept iff it lies within the reach of at least one target of
//      the group (one distance test per lane of the warp; union of the targets' spheres).
// Reach: density  r < h_build,i (list valid for every h <= h_build in the Newton iteration);
//        force    r < max(h_i, h_j) with the final h.
// List entry: (periodic image code << 27) | source index (cell order); image code
// c = cx + 3 cy + 9 cz, c_a = 0 none, 1 source shifted by -L_a, 2 by +L_a.
#pragma once
#include "build.cuh"

#define WALK_WARPS 8
#define WALK_STACK 160
#define WALK_TAKE 32    // a node holding <= WALK_TAKE particles is swept whole (no descent)

struct WalkParams {
  const int4* groups;
  int nsel;                 // groups to walk
  const int* sel;           // their ids (null: 0..nsel-1)
  const float4* xh;         // cell-order positions
  const float* reach;       // per particle: density h_build; force h (targets and sources)
  const uint32_t* perm;     // cell order -> caller index; targets are perm < n_own
  int64_t n_own;
  NodeArrays N;
  LevelGeom g;
  const int* topmap;
  const SortEntry* sorted;
  int force;
  float reach_max;          // max reach over all particles (force: source reach bound)
  float slack;              // absolute slack of the geometric tests (fp32 rounding)
  int64_t* off;             // per group: list offset (FILL reads)
  int* len;                 // per group: list length (COUNT writes)
  int* len_sel;             // per selected group: list length (COUNT writes, for the scan)
  uint32_t* out;            // list pool (FILL)
  unsigned long long* ctr;
};

#define WALK_CAP 384    // frontier entries (node | image code << 27), LIFO
#define WALK_DFS 112    // room for the depth-first fallback above the frontier
#define WALK_RQ 64      // queued leaf ranges streamed together
struct WalkSmem {
  int stk[WALK_CAP + WALK_DFS];
  int rq_first[WALK_RQ];
  int rq_code[WALK_RQ];
  int rq_pre[WALK_RQ + 1];  // exclusive prefix of the queued ranges' counts
  float4 s[32];             // staged box survivors: shifted position, reach
};

struct WalkState {
  float3 lo, hi;            // targets' bounding box
  float R;                  // max target reach
  float xi, yi, zi, ri;     // this lane's target (ri = -1: not a target)
  int64_t base;             // FILL: list offset of the group
  int cur;                  // entries emitted so far
};

__device__ __forceinline__ float reach_eff(float r, float slack) { return fmaf(r, 1.00001f, slack); }

// one chunk of <= 32 candidate sources (one per lane): keep those within reach of a target
template <bool FILL>
__device__ __forceinline__ void emit_chunk(const WalkParams& P, WalkState& W, WalkSmem& S, bool valid, int j,
                                           float px, float py, float pz, float hj, int code, int lane) {
  // 1. box filter against the targets' bounding box
  bool keep = false;
  if (valid) {
    const float ex = fmaxf(fmaxf(W.lo.x - px, px - W.hi.x), 0.f);
    const float ey = fmaxf(fmaxf(W.lo.y - py, py - W.hi.y), 0.f);
    const float ez = fmaxf(fmaxf(W.lo.z - pz, pz - W.hi.z), 0.f);
    const float rr = reach_eff(P.force ? fmaxf(W.R, hj) : W.R, P.slack);
    keep = fmaf(ex, ex, fmaf(ey, ey, ez * ez)) < rr * rr;
  }
  const unsigned bal = __ballot_sync(FULL_MASK, keep);
  if (!bal) return;
  const int m = __popc(bal);
  const int pos = __popc(bal & lanemask_lt());
  if (keep) S.s[pos] = make_float4(px, py, pz, P.force ? reach_eff(hj, P.slack) : 0.f);
  __syncwarp();
  // 2. union of the targets' spheres: lane = target, tests every staged survivor
  unsigned hm = 0u;
  if (W.ri >= 0.f) {
    const float ri = reach_eff(W.ri, P.slack);
    const float ri2 = ri * ri;
    for (int t = 0; t < m; ++t) {
      const float4 q = S.s[t];
      const float dx = W.xi - q.x, dy = W.yi - q.y, dz = W.zi - q.z;
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float lim2 = P.force ? fmaxf(ri2, q.w * q.w) : ri2;
      hm |= (unsigned)(r2 < lim2) << t;
    }
  }
  const unsigned km = __reduce_or_sync(FULL_MASK, hm);
  __syncwarp();
  const bool mine = keep && ((km >> pos) & 1u);
  const unsigned b2 = __ballot_sync(FULL_MASK, mine);
  if (FILL && mine)
    P.out[W.base + W.cur + __popc(b2 & lanemask_lt())] = ((uint32_t)code << SPH_IDX_BITS) | (uint32_t)j;
  W.cur += __popc(b2);
}

// shifted source position in the group's frame: x + k L (k in {-1, 0, 1} per axis)
__device__ __forceinline__ float3 shifted(float4 p, int code, const LevelGeom& g) {
  const int cx = code % 3, cy = (code / 3) % 3, cz = code / 9;
  return make_float3(cx == 1 ? p.x - g.L[0] : (cx == 2 ? p.x + g.L[0] : p.x),
                     cy == 1 ? p.y - g.L[1] : (cy == 2 ? p.y + g.L[1] : p.y),
                     cz == 1 ? p.z - g.L[2] : (cz == 2 ? p.z + g.L[2] : p.z));
}
__device__ __forceinline__ float shift_of(int c, float L) { return c == 1 ? -L : (c == 2 ? L : 0.f); }

// node box (group frame) within reach of the targets' box
__device__ __forceinline__ bool node_in_reach(const WalkParams& P, const WalkState& W, int node, int code) {
  const int4 c = P.N.ijk[node];
  const int l = c.w;
  const float sx = shift_of(code % 3, P.g.L[0]), sy = shift_of((code / 3) % 3, P.g.L[1]),
              sz = shift_of(code / 9, P.g.L[2]);
  const float cx = node_corner(c.x, l, 0, P.g) + sx, cy = node_corner(c.y, l, 1, P.g) + sy,
              cz = node_corner(c.z, l, 2, P.g) + sz;
  const float gx = fmaxf(fmaxf(cx - W.hi.x, W.lo.x - (cx + P.g.E[l][0])), 0.f);
  const float gy = fmaxf(fmaxf(cy - W.hi.y, W.lo.y - (cy + P.g.E[l][1])), 0.f);
  const float gz = fmaxf(fmaxf(cz - W.hi.z, W.lo.z - (cz + P.g.E[l][2])), 0.f);
  const float rr = reach_eff(P.force ? fmaxf(W.R, P.N.hmax[node]) : W.R, P.slack);
  return fmaf(gx, gx, fmaf(gy, gy, gz * gz)) < rr * rr;
}

// sweep a reached leaf (or small node): sorted window sweep if the leaf has presorted
// lists and lies to one side of the group, else its whole contiguous range
template <bool FILL>
__device__ __forceinline__ void sweep_node(const WalkParams& P, WalkState& W, WalkSmem& S, int node, int code,
                                           int lane) {
  const int first = P.N.first[node], cnt = P.N.count[node];
  const int64_t soff = P.N.sortoff[node];
  int k = 13;
  float3 cnr;
  if (soff >= 0) {
    const int4 c = P.N.ijk[node];
    const int l = c.w;
    cnr = make_float3(node_corner(c.x, l, 0, P.g) + shift_of(code % 3, P.g.L[0]),
                      node_corner(c.y, l, 1, P.g) + shift_of((code / 3) % 3, P.g.L[1]),
                      node_corner(c.z, l, 2, P.g) + shift_of(code / 9, P.g.L[2]));
    const int ox = cnr.x > W.hi.x ? 1 : (cnr.x + P.g.E[l][0] < W.lo.x ? -1 : 0);
    const int oy = cnr.y > W.hi.y ? 1 : (cnr.y + P.g.E[l][1] < W.lo.y ? -1 : 0);
    const int oz = cnr.z > W.hi.z ? 1 : (cnr.z + P.g.E[l][2] < W.lo.z ? -1 : 0);
    k = (ox + 1) * 9 + (oy + 1) * 3 + (oz + 1);
  }
  if (k == 13) {                                   // whole range
    for (int b0 = 0; b0 < cnt; b0 += 32) {
      const int e = b0 + lane;
      const bool v = e < cnt;
      float3 ps = make_float3(0.f, 0.f, 0.f);
      float hj = 0.f;
      if (v) {
        ps = shifted(P.xh[first + e], code, P.g);
        hj = P.reach[first + e];
      }
      emit_chunk<FILL>(P, W, S, v, first + e, ps.x, ps.y, ps.z, hj, code, lane);
    }
    return;
  }
  // sorted sweep along canonical direction d; the leaf lies on the +d side of the group
  // (ascending keys, nearest first) or on the -d side (flip: descending)
  const int d = slot_dir(k);
  const bool flip = slot_flip(k);
  const float3 du = dir_unit(d);
  const SortEntry* __restrict__ list = P.sorted + soff + (int64_t)d * cnt;
  float pr = W.ri >= 0.f ? proj(W.xi - cnr.x, W.yi - cnr.y, W.zi - cnr.z, du) : (flip ? INFINITY : -INFINITY);
  pr = flip ? warp_min_f(pr) : warp_max_f(pr);
  const float win = reach_eff(P.force ? fmaxf(W.R, P.N.hmax[node]) : W.R, P.slack) + P.slack;
  const float lim = flip ? pr - win : pr + win;
  for (int b0 = 0; b0 < cnt; b0 += 32) {
    const int e = b0 + lane;
    bool v = e < cnt;
    int j = 0;
    if (v) {
      const SortEntry en = list[flip ? cnt - 1 - e : e];
      v = flip ? en.key > lim : en.key < lim;
      j = en.idx;
    }
    const unsigned inwin = __ballot_sync(FULL_MASK, v);
    float3 ps = make_float3(0.f, 0.f, 0.f);
    float hj = 0.f;
    if (v) {
      ps = shifted(P.xh[j], code, P.g);
      hj = P.reach[j];
    }
    emit_chunk<FILL>(P, W, S, v, j, ps.x, ps.y, ps.z, hj, code, lane);
    if (__popc(inwin) < min(32, cnt - b0)) break;  // early exit
  }
}

// stream the queued leaf ranges as one sequence, 32 sources per chunk
template <bool FILL>
__device__ __forceinline__ void flush_ranges(const WalkParams& P, WalkState& W, WalkSmem& S, int& nq, int lane) {
  if (nq == 0) return;
  const int total = S.rq_pre[nq];
  for (int b0 = 0; b0 < total; b0 += 32) {
    const int gi = b0 + lane;
    const bool v = gi < total;
    int j = 0, code = 0;
    float3 ps = make_float3(0.f, 0.f, 0.f);
    float hj = 0.f;
    if (v) {
      int r = 0;                                    // rq_pre[r] <= gi < rq_pre[r+1]
#pragma unroll
      for (int step = 32; step > 0; step >>= 1)
        if (r + step < nq && S.rq_pre[r + step] <= gi) r += step;
      j = S.rq_first[r] + (gi - S.rq_pre[r]);
      code = S.rq_code[r];
      ps = shifted(P.xh[j], code, P.g);
      hj = P.reach[j];
    }
    emit_chunk<FILL>(P, W, S, v, j, ps.x, ps.y, ps.z, hj, code, lane);
  }
  __syncwarp();
  nq = 0;
}

// depth-first descent of one subtree (fallback when the frontier is full)
template <bool FILL>
__device__ void dfs_subtree(const WalkParams& P, WalkState& W, WalkSmem& S, int* stk, int entry, int& nq, int lane) {
  if (lane == 0) stk[0] = entry;
  int top = 1;
  __syncwarp();
  while (top > 0) {
    const int e = stk[--top];
    __syncwarp();
    const int nd = e & SPH_IDX_MASK, code = (int)((unsigned)e >> SPH_IDX_BITS);
    const int4 rec = P.N.rec[nd];
    if (rec.z >= 0 && rec.y > WALK_TAKE) {
      int ch = -1;
      const int mask = rec.w & 0xff;
      if (lane < __popc(mask)) {
        ch = rec.z + lane;
        if (!node_in_reach(P, W, ch, code)) ch = -1;
      }
      const unsigned ok = __ballot_sync(FULL_MASK, ch >= 0);
      if (ch >= 0) stk[top + __popc(ok & lanemask_lt())] = ch | (code << SPH_IDX_BITS);
      top += __popc(ok);
      __syncwarp();
    } else {
      flush_ranges<FILL>(P, W, S, nq, lane);
      sweep_node<FILL>(P, W, S, nd, code, lane);
    }
  }
}

// Warp per group: the cells within reach, 32 nodes per round (each lane tests one node's
// box; reached internal nodes push their children, reached leaves queue their ranges),
// then the queued ranges streamed through the source filters.
template <bool FILL>
__global__ void __launch_bounds__(WALK_WARPS * 32) k_walk(WalkParams P) {
  __shared__ WalkSmem smem[WALK_WARPS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * WALK_WARPS + wib;
  if (w >= P.nsel) return;
  WalkSmem& S = smem[wib];
  const int gid = P.sel ? P.sel[w] : w;
  const int4 grp = P.groups[gid];
  const int s = grp.y + lane;
  WalkState W;
  W.ri = -1.f;
  W.xi = W.yi = W.zi = 0.f;
  if (lane < grp.z && P.perm[s] < (uint32_t)P.n_own) {
    const float4 p = P.xh[s];
    W.xi = p.x;
    W.yi = p.y;
    W.zi = p.z;
    W.ri = P.reach[s];
  }
  const bool tg = W.ri >= 0.f;
  W.lo = make_float3(warp_min_f(tg ? W.xi : INFINITY), warp_min_f(tg ? W.yi : INFINITY),
                     warp_min_f(tg ? W.zi : INFINITY));
  W.hi = make_float3(warp_max_f(tg ? W.xi : -INFINITY), warp_max_f(tg ? W.yi : -INFINITY),
                     warp_max_f(tg ? W.zi : -INFINITY));
  W.R = warp_max_f(tg ? W.ri : 0.f);
  W.cur = 0;
  W.base = FILL ? P.off[gid] : 0;
  int nq = 0;
  if (__any_sync(FULL_MASK, tg)) {
    // top cells (unwrapped indices) overlapping the box grown by the largest possible reach
    const float Rw = reach_eff(P.force ? fmaxf(W.R, P.reach_max) : W.R, P.slack) + P.slack;
    int a0[3], na[3];
    const float lo3[3] = {W.lo.x, W.lo.y, W.lo.z}, hi3[3] = {W.hi.x, W.hi.y, W.hi.z};
    int T = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float E = P.g.E[0][a];
      int lo_i = (int)floorf((lo3[a] - Rw) / E), hi_i = (int)floorf((hi3[a] + Rw) / E);
      lo_i = max(lo_i, -P.g.ntop[a]);
      hi_i = min(hi_i, 2 * P.g.ntop[a] - 1);
      a0[a] = lo_i;
      na[a] = hi_i - lo_i + 1;
      T *= na[a];
    }
    for (int tb = 0; tb < T; tb += 32) {
      // seed the frontier with this chunk's top cells (reach tested when popped)
      const int t = tb + lane;
      int ent = -1;
      if (t < T) {
        const int ux = a0[0] + t % na[0], uy = a0[1] + (t / na[0]) % na[1], uz = a0[2] + t / (na[0] * na[1]);
        const int nx = P.g.ntop[0], ny = P.g.ntop[1], nz = P.g.ntop[2];
        const int ix = ((ux % nx) + nx) % nx, iy = ((uy % ny) + ny) % ny, iz = ((uz % nz) + nz) % nz;
        const int kx = (ux - ix) / nx, ky = (uy - iy) / ny, kz = (uz - iz) / nz;   // -1, 0, 1
        const int code =
            (kx < 0 ? 1 : (kx > 0 ? 2 : 0)) + 3 * (ky < 0 ? 1 : (ky > 0 ? 2 : 0)) + 9 * (kz < 0 ? 1 : (kz > 0 ? 2 : 0));
        const int node = P.topmap[ix + (int64_t)nx * (iy + (int64_t)ny * iz)];
        if (node >= 0) ent = node | (code << SPH_IDX_BITS);
      }
      const unsigned sb = __ballot_sync(FULL_MASK, ent != -1);
      if (ent != -1) S.stk[__popc(sb & lanemask_lt())] = ent;
      int top = __popc(sb);
      __syncwarp();
      while (top > 0) {
        int k = min(32, top);
        while (k > 0 && top - k + 8 * k > WALK_CAP) --k;
        if (k == 0) {                                  // frontier full: one subtree depth-first
          const int e = S.stk[top - 1];
          __syncwarp();
          --top;
          dfs_subtree<FILL>(P, W, S, S.stk + top, e, nq, lane);
          continue;
        }
        int e = 0;
        if (lane < k) e = S.stk[top - k + lane];
        __syncwarp();
        top -= k;
        const int nd = e & SPH_IDX_MASK, code = (int)((unsigned)e >> SPH_IDX_BITS);
        bool reach = false, leaf = false, srt = false;
        int4 rec = make_int4(0, 0, -1, 0);
        if (lane < k) {
          rec = P.N.rec[nd];
          reach = node_in_reach(P, W, nd, code);
          leaf = reach && !(rec.z >= 0 && rec.y > WALK_TAKE);
          srt = leaf && P.N.sortoff[nd] >= 0;
        }
        // reached internal nodes push their children
        const int nch = (reach && !leaf) ? __popc(rec.w & 0xff) : 0;
        int pre = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL_MASK, pre, o);
          if (lane >= o) pre += y;
        }
        const int tot = __shfl_sync(FULL_MASK, pre, 31);
        for (int c2 = 0; c2 < nch; ++c2) S.stk[top + pre - nch + c2] = (rec.z + c2) | (code << SPH_IDX_BITS);
        top += tot;
        // reached unsorted leaves: queue their ranges
        const bool ql = leaf && !srt;
        const unsigned qb = __ballot_sync(FULL_MASK, ql);
        if (nq + __popc(qb) > WALK_RQ) flush_ranges<FILL>(P, W, S, nq, lane);
        if (ql) {
          const int q = nq + __popc(qb & lanemask_lt());
          S.rq_first[q] = rec.x;
          S.rq_code[q] = code;
          S.rq_pre[q + 1] = rec.y;                  // counts; prefix below
        }
        __syncwarp();
        if (qb) {
          const int nn = nq + __popc(qb);
          if (lane == 0) S.rq_pre[0] = 0;
          __syncwarp();
          // exclusive prefix over the queue (<= 64 entries): lanes own entries lane, lane+32
          int c0 = (lane + 1 <= nn && lane >= nq) ? S.rq_pre[lane + 1] : 0;
          int c1 = (lane + 33 <= nn && lane + 32 >= nq) ? S.rq_pre[lane + 33] : 0;
          __syncwarp();
          // recompute the whole prefix from the raw counts of the new entries
          int v0 = c0, v1 = c1;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y0 = __shfl_up_sync(FULL_MASK, v0, o), y1 = __shfl_up_sync(FULL_MASK, v1, o);
            if (lane >= o) {
              v0 += y0;
              v1 += y1;
            }
          }
          const int t0 = __shfl_sync(FULL_MASK, v0, 31);
          const int basep = S.rq_pre[nq];
          __syncwarp();
          if (lane >= nq && lane + 1 <= nn) S.rq_pre[lane + 1] = basep + v0;
          if (lane + 32 >= nq && lane + 33 <= nn) S.rq_pre[lane + 33] = basep + t0 + v1;
          __syncwarp();
          nq = nn;
        }
        // reached sorted leaves: windowed sweeps, one at a time
        unsigned sbm = __ballot_sync(FULL_MASK, srt);
        while (sbm) {
          const int src = __ffs(sbm) - 1;
          sbm &= sbm - 1;
          const int snd = __shfl_sync(FULL_MASK, nd, src), scode = __shfl_sync(FULL_MASK, code, src);
          sweep_node<FILL>(P, W, S, snd, scode, lane);
        }
      }
    }
    flush_ranges<FILL>(P, W, S, nq, lane);
  }
  if (!FILL && lane == 0) {
    P.len[gid] = W.cur;
    if (P.len_sel) P.len_sel[w] = W.cur;
  }
  if (FILL && lane == 0 && W.cur != P.len[gid]) atomicOr(&P.ctr[C_ERR], 1ull << 20);   // count/fill mismatch
}

// list offsets of the selected groups: base + exclusive scan of their lengths
__global__ void k_set_offsets(int nsel, const int* __restrict__ sel, const int64_t* __restrict__ scan, int64_t base,
                              int64_t* __restrict__ off) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nsel) return;
  off[sel ? sel[w] : w] = base + scan[w];
}

// groups flagged for a list rebuild (a target's h outgrew its h_build), compaction flags
#define HS_DONE 0
#define HS_ACTIVE 1
#define HS_REGROW 2   // active; h_build grown: its group's density list is rebuilt before the next pass
__global__ void k_group_flags(const int4* __restrict__ groups, int ngroups, uint8_t* __restrict__ state,
                              int* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int gi = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (gi >= ngroups) return;
  const int4 g = groups[gi];
  bool r = false;
  if (lane < g.z) {
    const int s = g.y + lane;
    r = state[s] == HS_REGROW;
    if (r) state[s] = HS_ACTIVE;
  }
  const bool any = __any_sync(FULL_MASK, r);
  if (lane == 0) flag[gi] = any ? 1 : 0;
}

__global__ void k_compact_idx(const int* __restrict__ flag, const int* __restrict__ scan, int64_t n,
                              int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[scan[i]] = (int32_t)i;
}

__global__ void k_widen_i32(const int* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}
