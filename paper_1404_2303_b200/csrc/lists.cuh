// lists.cuh — neighbour finding: the tree walk that builds the interaction lists
// (section 3.2-3.3).
//
// The paper finds the interacting pairs through cell pairs: every particle sits in a cell
// whose edge is at least its h, so its partners lie in the 26 neighbouring cells
// (P:471-499); pairs of large cells are refined into pairs of their children;
// and the particles of the two cells of a pair are swept in the order of their projection
// onto the axis joining the cells, so the sweep stops at the first particle whose projected
// distance exceeds h (P:644-698, 13 presorted directions per cell).
//
// On the GPU the same search runs per target group (<= 32 consecutive particles of one
// cell, one warp) and its result is stored, so the h iteration and the two interaction
// loops reuse it (the paper reuses its sorts for both loops):
//   1. the cells within reach of the group: the top cells around the group's bounding box
//      (with their periodic images), refined into their children while a
//      child's box is within reach (the pair refinement of P:523-532, decided per child box
//      instead of per cell pair), 32 cells per round (one per lane);
//   2. in a reached leaf the sources are swept in the leaf's presorted order along the
//      canonical direction joining the group and the leaf, stopping at the first source
//      whose projection lies beyond the window (the sorted sweep of P:644-669, R6, R20);
//      leaves without presorted lists are streamed whole, 32 sources per chunk;
//   3. each swept source passes a box test against the group, then one exact distance test
//      per target (lane), and is recorded:
//        NB mode    per target i, the squared distances r^2 < h_build,i^2 (the neighbour
//                   lists of the h iteration, k_hsolve);
//        UNION mode per group, the sources within reach of at least one target, with
//                   reach max(h_i, h_j) at the final h: the list the density and
//                   force loops stream (interact.cuh). Counted, then filled.
// Coordinates are relative to the group's first particle o with exact periodic images
// (rel_pos), so the recorded r^2 are the ones the interaction kernels compute.
// UNION entry: (periodic image code << 27) | source index (cell order); image code
// c = cx + 3 cy + 9 cz, c_a = 0 none, 1 source at x - L_a, 2 source at x + L_a.
#pragma once
#include "build.cuh"
#include "hiter.cuh"

#ifndef WALK_WARPS
#define WALK_WARPS 2
#endif
#ifndef WALK_TAKE
#define WALK_TAKE 64    // a node holding <= WALK_TAKE particles is swept whole (no descent; 32: +0.08 ms, 128: +0.08)
#endif
#ifndef WALK_CAP
#define WALK_CAP 384    // frontier entries (node | image code << 27), LIFO
#endif
#ifndef WALK_DFS
#define WALK_DFS 112    // room for the depth-first fallback above the frontier
#endif
#ifndef WALK_RQ
#define WALK_RQ 64      // queued leaf ranges streamed together
#endif
#ifndef SPH_INWALK_PASSES
#define SPH_INWALK_PASSES 6   // NB walk passes per group and launch (re-walks without a host round)
#endif
#ifndef NB_ROWS
#define NB_ROWS 1       // neighbour-list slab: one contiguous row of K per particle (0: column-interleaved per group)
#endif
#ifndef NB_PREFETCH
#define NB_PREFETCH 1   // prefetch each neighbour-list row into L1 before the h sums
#endif
#ifndef SPHERE_HINT
#define SPHERE_HINT 1   // interaction-list walk: test first the target that reached the node's parent
#endif
#ifndef UNION_PACKED
#define UNION_PACKED 1  // interaction-list walk: packed FP32 pair tests (tools/sweep.sh)
#endif
#ifndef RANGE_MASK
#define RANGE_MASK 1
#endif
#ifndef SPHERE_VOTE
#define SPHERE_VOTE 4   // node-vs-target-sphere tests between warp votes for an early exit
#endif

#define MODE_NB 0
#define MODE_COUNT 1
#define MODE_FILL 2

#ifdef SPH_WALK_STATS
// instrumentation (build with -DSPH_WALK_STATS; printed by sph_build_cells): per NB-walk pass,
// [0] warp passes, [1] active target lanes, [2] staged box survivors (warp level),
// [3] recorded entries, [4] staged chunks
__device__ unsigned long long g_walkstats[8][5];
#endif

// source position relative to the group origin o (oL = o - L), periodic image code c:
// x - L is exact for a source near L, o - L for a group near L (Sterbenz; R19, H2)
__device__ __forceinline__ float3 rel_pos(float4 p, uint32_t code, float3 o, float3 oL, const float* L) {
  const int cx = code % 3, cy = (code / 3) % 3, cz = code / 9;
  const float x = (cx == 1 ? p.x - L[0] : p.x) - (cx == 2 ? oL.x : o.x);
  const float y = (cy == 1 ? p.y - L[1] : p.y) - (cy == 2 ? oL.y : o.y);
  const float z = (cz == 1 ? p.z - L[2] : p.z) - (cz == 2 ? oL.z : o.z);
  return make_float3(x, y, z);
}
__device__ __forceinline__ float shift_of(int c, float L) { return c == 1 ? -L : (c == 2 ? L : 0.f); }
__device__ __forceinline__ float reach_eff(float r, float slack) { return fmaf(r, 1.00001f, slack); }

struct WalkParams {
  const int4* groups;
  int nsel;                 // groups to walk
  const int* sel;           // their ids (null: 0..nsel-1)
  const int* nsel_dev;      // if set: the number of groups in sel (device; nsel is a bound)
  int* rg_out;              // if set: groups with a lane left in HS_REGROW are appended here
  int* rg_cnt;              //   (count, atomic; order is scheduling only, results do not depend on it)
  const uint8_t* tgt;       // cell order: 1 = target (owned and active), 0 = source only
  unsigned long long* raw_out;  // if set: sources streamed through the filters, summed (SPH_F_COUNT_CANDIDATES)
  const float4* xh;         // cell-order positions
  const float* reach;       // per particle: NB h_build; UNION the h used for the reach (0: none)
  int reach_xhw;            // UNION: reach[j] == xh[j].w for every particle (no halo): read it from the position record
  const uint8_t* tsel;      // NB: targets are the particles with tsel == tsel_val (null: owned)
  uint8_t tsel_val;
  const uint32_t* perm;     // cell order -> caller index; targets are owned (perm < n_own)
  int64_t n_own;
  NodeArrays N;
  LevelGeom g;
  const int* topmap;
  const SortEntry* sorted;
  int any_sorted;           // some leaf has presorted lists (else no sortoff is read)
  float reach_max;          // UNION: max source reach (bound for the top-cell range)
  const unsigned long long* reach_max_bits;   // if set: reach_max as float bits on the device
  float slack;              // absolute slack of the box tests (fp32 rounding of corners)
  // UNION
  int64_t* off;             // per group: list offset (FILL reads)
  int* len;                 // per group: list length (COUNT writes)
  int* len_sel;             // per selected group: list length (COUNT writes, for the scan)
  uint32_t* out;            // list pool (FILL)
  int ucap;                 // FILL: entries recorded per group (beyond: counted only)
  int check;                // FILL: 1 = second pass into exact space, verify the length
  // NB
  float* nb_r2;             // [n * K]: particle s's entries (r, or r^2 if !NB_STORE_R; hiter.cuh), row s (NB_ROWS)
  int* nb_cnt;              // [n] sources with r^2 < h_build^2 (may exceed K: overflow)
  int K;
  unsigned long long* nb_entries;   // NB: running total of recorded entries
  // NB + solve: the h iteration runs in the walk's epilogue on the list just recorded
  int solve;
  float* hb_w;              // h_build (== reach), written back
  float *lo, *hi;           // Newton brackets
  uint8_t* state;
  uint8_t* shrunk;          // first overflow seen
  int64_t* ovf_cnt;         // repeat overflow: exact count (pool)
  int64_t* ovf_off_w;       // -1: the list is in the slab
  unsigned long long* hc;   // solve counters (HC_*)
  float n_t, tol, margin, hcap;
  int max_iter;
  const int64_t* ovf_off;   // NB overflow walk: the particle's list at ovf + ovf_off[s] (contiguous)
  float* ovf;
  unsigned long long* ctr;
};

struct WalkSmem {
  int stk[WALK_CAP + WALK_DFS];
  uint8_t hint[WALK_CAP];   // per frontier entry: a target that reached the parent
  int rq_first[WALK_RQ];
  int rq_code[WALK_RQ];
  float4 rq_so[WALK_RQ];    // per queued range: source pre-shift (x - L for a source near L)
  float4 rq_oo[WALK_RQ];    //   and the origin it is taken relative to (o, or o - L)
  float4 shf[27];           // image code -> shift vector
  int rq_pre[WALK_RQ + 1];  // exclusive prefix of the queued ranges' counts
  float4 s[32];             // staged box survivors: relative position, source reach
  float4 tgt[32];           // the targets' spheres (relative position, reach), compacted
};

struct WalkState {
  float3 o, oL;             // group origin, origin - L
  float3 lo, hi;            // targets' bounding box (relative)
  float R;                  // max target reach
  float xi, yi, zi, ri;     // this lane's target (relative; ri = -1: not a target)
  int64_t base;             // FILL: list offset of the group / NB: column base
  int cur;                  // UNION: entries emitted so far; NB: this lane's count
  int gz, lane;
  int raw;                  // sources streamed through the filters (diagnostics)
  int ntg;                  // targets (staged in WalkSmem::tgt)
#ifdef SPH_WALK_STATS
  long long st_surv, st_calls;
#endif
  bool spheres;             // refine node tests by the individual targets' spheres
};

// one chunk of <= 32 candidate sources (one per lane, relative position p, reach hj)
template <int MODE>
__device__ __forceinline__ void emit_chunk(const WalkParams& P, WalkState& W, WalkSmem& S, bool valid, int j,
                                           float3 p, float hj, int code) {
  const int lane = W.lane;
  // 1. box filter against the targets' bounding box
  bool keep = false;
  if (valid) {
    const float ex = fmaxf(fmaxf(W.lo.x - p.x, p.x - W.hi.x), 0.f);
    const float ey = fmaxf(fmaxf(W.lo.y - p.y, p.y - W.hi.y), 0.f);
    const float ez = fmaxf(fmaxf(W.lo.z - p.z, p.z - W.hi.z), 0.f);
    const float rr = reach_eff(MODE == MODE_NB ? W.R : fmaxf(W.R, hj), P.slack);
    keep = fmaf(ex, ex, fmaf(ey, ey, ez * ez)) < rr * rr;
  }
  W.raw += __popc(__ballot_sync(FULL_MASK, valid));
  const unsigned bal = __ballot_sync(FULL_MASK, keep);
  if (!bal) return;
  const int m = __popc(bal);
#ifdef SPH_WALK_STATS
  if (MODE == MODE_NB) {
    W.st_surv += m;
    W.st_calls += 1;
  }
#endif
  const int pos = __popc(bal & lanemask_lt());
#if UNION_PACKED
  if (MODE != MODE_NB) {
    // SoA planes x, y, z, reach^2 for packed FP32 pair tests; an odd count is padded with a
    // far source
    float* sx = reinterpret_cast<float*>(S.s);
    if (keep) {
      const float w = reach_eff(hj, 0.f);
      sx[pos] = p.x;
      sx[32 + pos] = p.y;
      sx[64 + pos] = p.z;
      sx[96 + pos] = w * w;
    }
    if (lane == 0 && (m & 1)) {
      sx[m] = sx[32 + m] = sx[64 + m] = 1e30f;
      sx[96 + m] = 0.f;
    }
  } else
#endif
  if (keep) S.s[pos] = make_float4(p.x, p.y, p.z, MODE == MODE_NB ? 0.f : reach_eff(hj, 0.f));
  __syncwarp();
  // 2. exact distance test per target (lane)
  if (MODE == MODE_NB) {
    if (W.ri >= 0.f) {
      const float ri = reach_eff(W.ri, 0.f);
      const float ri2 = ri * ri;
      // the pool list and the slab rows are contiguous, the slab columns (!NB_ROWS) strided by gz
      const int step = (P.ovf || NB_ROWS) ? 1 : W.gz;
      const int lim = P.ovf ? INT_MAX : P.K;
      float* wp = P.ovf ? P.ovf + W.base + W.cur : P.nb_r2 + W.base + (int64_t)W.cur * step;
      int cur = W.cur;
      for (int t = 0; t < m; ++t) {
        const float4 q = S.s[t];
        const float dx = W.xi - q.x, dy = W.yi - q.y, dz = W.zi - q.z;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        // every lane computes the entry, the store and the pointer step are predicated: no
        // reconvergence block per source (the hits diverge across the warp)
        const float e = nb_stored(r2);
        const bool hit = r2 < ri2;
        if (hit && cur < lim) *wp = e;
        wp += hit ? step : 0;
        cur += hit ? 1 : 0;
      }
      W.cur = cur;
    }
    __syncwarp();
    return;
  }
  unsigned hm = 0u;
  if (W.ri >= 0.f) {
    const float ri = reach_eff(W.ri, 0.f);
    const float ri2 = ri * ri;
#if UNION_PACKED
    // two sources per packed instruction, the interaction kernels' r^2 operation order
    const float2* X2 = reinterpret_cast<const float2*>(S.s);
    const float2* Y2 = X2 + 16;
    const float2* Z2 = X2 + 32;
    const float2* R2 = X2 + 48;
    for (int t = 0; t < (m + 1) >> 1; ++t) {
      const float2 r2 = r2_pair(W.xi, W.yi, W.zi, X2[t], Y2[t], Z2[t]);
      const float2 w2 = R2[t];
      hm |= ((unsigned)(r2.x < fmaxf(ri2, w2.x)) | ((unsigned)(r2.y < fmaxf(ri2, w2.y)) << 1)) << (2 * t);
    }
#else
    for (int t = 0; t < m; ++t) {
      const float4 q = S.s[t];
      const float dx = W.xi - q.x, dy = W.yi - q.y, dz = W.zi - q.z;
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      hm |= (unsigned)(r2 < fmaxf(ri2, q.w * q.w)) << t;
    }
#endif
  }
  const unsigned km = __reduce_or_sync(FULL_MASK, hm);
  __syncwarp();
  const bool mine = keep && ((km >> pos) & 1u);
  const unsigned b2 = __ballot_sync(FULL_MASK, mine);
  if (MODE == MODE_FILL && mine) {
    const int idx = W.cur + __popc(b2 & lanemask_lt());
    if (idx < P.ucap) P.out[W.base + idx] = ((uint32_t)code << SPH_IDX_BITS) | (uint32_t)j;
  }
  W.cur += __popc(b2);
}

// node box corner in the group's frame (fp32; the box tests carry an absolute slack)
__device__ __forceinline__ float3 node_corner_rel(const WalkParams& P, const WalkState& W, const WalkSmem& S, int4 c,
                                                  int code) {
  const int l = c.w;
  const float4 sh = S.shf[code];
  return make_float3(fmaf((float)c.x, P.g.E[l][0], sh.x) - W.o.x, fmaf((float)c.y, P.g.E[l][1], sh.y) - W.o.y,
                     fmaf((float)c.z, P.g.E[l][2], sh.z) - W.o.z);
}

// node box within reach of the targets' box
template <int MODE>
__device__ __forceinline__ bool node_in_reach(const WalkParams& P, const WalkState& W, const WalkSmem& S, int node,
                                              int code) {
  const int4 c = P.N.ijk[node];
  const int l = c.w;
  const float3 cr = node_corner_rel(P, W, S, c, code);
  const float gx = fmaxf(fmaxf(cr.x - W.hi.x, W.lo.x - (cr.x + P.g.E[l][0])), 0.f);
  const float gy = fmaxf(fmaxf(cr.y - W.hi.y, W.lo.y - (cr.y + P.g.E[l][1])), 0.f);
  const float gz = fmaxf(fmaxf(cr.z - W.hi.z, W.lo.z - (cr.z + P.g.E[l][2])), 0.f);
  const float rr = reach_eff(MODE == MODE_NB ? W.R : fmaxf(W.R, P.N.hmax[node]), P.slack);
  return fmaf(gx, gx, fmaf(gy, gy, gz * gz)) < rr * rr;
}

// Refines the box test: the node (one per lane) is kept iff its box is within reach of at
// least one target's own sphere (each target broadcast in turn), so a group whose targets'
// h differ widely does not visit the cells only its bounding box reaches.
// hint: a target that reached the node's parent (tested first; children usually meet the
// same target); *first_hit returns the target that reached this node, for its children.
template <int MODE>
__device__ __forceinline__ bool node_in_spheres(const WalkParams& P, const WalkState& W, const WalkSmem& S, int node,
                                                int code, bool coarse, int hint = 0, int* first_hit = nullptr) {
  if (!W.spheres || !__any_sync(FULL_MASK, coarse)) return coarse;
  float3 lo = make_float3(0.f, 0.f, 0.f), hi = lo;
  float hmn = 0.f;
  if (coarse) {
    const int4 c = P.N.ijk[node];
    lo = node_corner_rel(P, W, S, c, code);
    hi = make_float3(lo.x + P.g.E[c.w][0], lo.y + P.g.E[c.w][1], lo.z + P.g.E[c.w][2]);
    if (MODE != MODE_NB) hmn = P.N.hmax[node];
  }
  bool hit = false;
  int ht = 0;
#if SPHERE_HINT
  if (MODE != MODE_NB) {
    const float4 q = S.tgt[min(hint, W.ntg - 1)];
    const float gx = fmaxf(fmaxf(lo.x - q.x, q.x - hi.x), 0.f);
    const float gy = fmaxf(fmaxf(lo.y - q.y, q.y - hi.y), 0.f);
    const float gz = fmaxf(fmaxf(lo.z - q.z, q.z - hi.z), 0.f);
    const float rr = MODE == MODE_NB ? q.w : fmaxf(q.w, reach_eff(hmn, P.slack));
    hit = fmaf(gx, gx, fmaf(gy, gy, gz * gz)) < rr * rr;
    ht = min(hint, W.ntg - 1);
  }
  if (MODE == MODE_NB || !__all_sync(FULL_MASK, hit || !coarse))
#endif
  for (int t0 = 0; t0 < W.ntg; t0 += SPHERE_VOTE) {
#pragma unroll
    for (int k = 0; k < SPHERE_VOTE; ++k) {
      const int t = min(t0 + k, W.ntg - 1);   // (a repeated last target is harmless)
      const float4 q = S.tgt[t];
      const float gx = fmaxf(fmaxf(lo.x - q.x, q.x - hi.x), 0.f);
      const float gy = fmaxf(fmaxf(lo.y - q.y, q.y - hi.y), 0.f);
      const float gz = fmaxf(fmaxf(lo.z - q.z, q.z - hi.z), 0.f);
      const float rr = MODE == MODE_NB ? q.w : fmaxf(q.w, reach_eff(hmn, P.slack));
      const bool h = fmaf(gx, gx, fmaf(gy, gy, gz * gz)) < rr * rr;
      if (MODE != MODE_NB && h && !hit) ht = t;
      hit |= h;
    }
    if (__all_sync(FULL_MASK, hit || !coarse)) break;   // every kept node already hit
  }
  if (first_hit) *first_hit = ht;
  return coarse && hit;
}

// sorted window sweep of a leaf with presorted lists that lies to one side of the group,
// else its whole contiguous range
template <int MODE>
__device__ __forceinline__ void sweep_node(const WalkParams& P, WalkState& W, WalkSmem& S, int node, int code) {
  const int lane = W.lane;
  const int first = P.N.first[node], cnt = P.N.count[node];
  const int64_t soff = P.any_sorted ? P.N.sortoff[node] : -1;
  const float* L = P.g.L;
  int k = 13;
  float3 cr = make_float3(0.f, 0.f, 0.f);
  if (soff >= 0) {
    const int4 c = P.N.ijk[node];
    const int l = c.w;
    cr = node_corner_rel(P, W, S, c, code);
    const int ox = cr.x > W.hi.x ? 1 : (cr.x + P.g.E[l][0] < W.lo.x ? -1 : 0);
    const int oy = cr.y > W.hi.y ? 1 : (cr.y + P.g.E[l][1] < W.lo.y ? -1 : 0);
    const int oz = cr.z > W.hi.z ? 1 : (cr.z + P.g.E[l][2] < W.lo.z ? -1 : 0);
    k = (ox + 1) * 9 + (oy + 1) * 3 + (oz + 1);
  }
  if (k == 13) {
    for (int b0 = 0; b0 < cnt; b0 += 32) {
      const int e = b0 + lane;
      const bool v = e < cnt;
      float3 p = make_float3(0.f, 0.f, 0.f);
      float hj = 0.f;
      if (v) {
        const float4 q = P.xh[first + e];
        p = rel_pos(q, code, W.o, W.oL, L);
        hj = P.reach_xhw ? q.w : P.reach[first + e];
      }
      emit_chunk<MODE>(P, W, S, v, first + e, p, hj, code);
    }
    return;
  }
  // the leaf lies on the +d side of the group (ascending keys, nearest first) or on the
  // -d side (flip: descending)
  const int d = slot_dir(k);
  const bool flip = slot_flip(k);
  const float3 du = dir_unit(d);
  const SortEntry* __restrict__ list = P.sorted + soff + (int64_t)d * cnt;
  float pr = W.ri >= 0.f ? proj(W.xi - cr.x, W.yi - cr.y, W.zi - cr.z, du) : (flip ? INFINITY : -INFINITY);
  pr = flip ? warp_min_f(pr) : warp_max_f(pr);
  const float win = reach_eff(MODE == MODE_NB ? W.R : fmaxf(W.R, P.N.hmax[node]), P.slack) + P.slack;
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
    float3 p = make_float3(0.f, 0.f, 0.f);
    float hj = 0.f;
    if (v) {
      const float4 q = P.xh[j];
      p = rel_pos(q, code, W.o, W.oL, L);
      hj = P.reach_xhw ? q.w : P.reach[j];
    }
    emit_chunk<MODE>(P, W, S, v, j, p, hj, code);
    if (__popc(inwin) < min(32, cnt - b0)) break;   // early exit
  }
}

// stream the queued leaf ranges as one sequence, 32 sources per chunk
template <int MODE>
__device__ __forceinline__ void flush_ranges(const WalkParams& P, WalkState& W, WalkSmem& S, int& nq) {
  if (nq == 0) return;
  const int lane = W.lane;
  const int total = S.rq_pre[nq];
  int rs = 0;                                       // the range holding b0
  // lane gi = b0 + lane of a chunk: its range r and source j (range starts inside [b0, b0 + 32)
  // as a bit mask: queued ranges are never empty, so starts are distinct; lane gi lies in range
  // rs + #{starts <= gi})
  auto locate = [&](int b0, int& r, int& j, bool& v) {
    const int gi = b0 + lane;
    v = gi < total;
#if RANGE_MASK
    unsigned bm = 0u;
    if (rs + 1 + lane < nq) {
      const int B = S.rq_pre[rs + 1 + lane];
      if (B < b0 + 32) bm = 1u << (B - b0);
    }
    bm = __reduce_or_sync(FULL_MASK, bm);
    r = rs + __popc(bm & (lanemask_lt() | (1u << lane)));
    rs += __popc(bm);
#else
    r = 0;                                        // rq_pre[r] <= gi < rq_pre[r+1]
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)
      if (r + step < nq && S.rq_pre[r + step] <= gi) r += step;
#endif
    j = v ? S.rq_first[r] + (gi - S.rq_pre[r]) : 0;
  };
  for (int b0 = 0; b0 < total; b0 += 32) {
    int r, j;
    bool v;
    locate(b0, r, j, v);
    int code = 0;
    float3 p = make_float3(0.f, 0.f, 0.f);
    float hj = 0.f;
    if (v) {
      code = S.rq_code[r];
      const float4 q = P.xh[j], so = S.rq_so[r], oo = S.rq_oo[r];
      p = make_float3((q.x + so.x) - oo.x, (q.y + so.y) - oo.y, (q.z + so.z) - oo.z);
      hj = P.reach_xhw ? q.w : P.reach[j];
    }
    emit_chunk<MODE>(P, W, S, v, j, p, hj, code);
  }
  __syncwarp();
  nq = 0;
}

// depth-first descent of one subtree (fallback when the frontier is full)
template <int MODE>
__device__ void dfs_subtree(const WalkParams& P, WalkState& W, WalkSmem& S, int* stk, int entry, int& nq) {
  const int lane = W.lane;
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
      bool rc = false;
      if (lane < __popc(rec.w & 0xff)) {
        ch = rec.z + lane;
        rc = node_in_reach<MODE>(P, W, S, ch, code);
      }
      rc = node_in_spheres<MODE>(P, W, S, ch, code, rc);
      if (!rc) ch = -1;
      const unsigned ok = __ballot_sync(FULL_MASK, ch >= 0);
      if (ch >= 0) stk[top + __popc(ok & lanemask_lt())] = ch | (code << SPH_IDX_BITS);
      top += __popc(ok);
      __syncwarp();
    } else {
      flush_ranges<MODE>(P, W, S, nq);
      sweep_node<MODE>(P, W, S, nd, code);
    }
  }
}

// Warp per group: the cells within reach, 32 nodes per round (each lane tests one node's
// box; reached internal nodes push their children, reached leaves queue their ranges),
// and the queued ranges streamed through the source filters.
template <int MODE>
#ifndef WALK_MINB
#define WALK_MINB 0     // min resident blocks for __launch_bounds__ (0: none; register use is then the compiler's)
#endif
#ifndef WALK_MAXNREG
#define WALK_MAXNREG 72   // pinned: left free, ptxas flips k_walk<NB> between 72 (small spills) and 96
                          // registers on unrelated edits, and 96 costs 0.5 ms (21 instead of 28 warps/SM)
#endif
#if WALK_MAXNREG > 0
#define WALK_BOUNDS __maxnreg__(WALK_MAXNREG)
#elif WALK_MINB > 0
#define WALK_BOUNDS __launch_bounds__(WALK_WARPS * 32, WALK_MINB)
#else
#define WALK_BOUNDS __launch_bounds__(WALK_WARPS * 32)
#endif
__global__ void WALK_BOUNDS k_walk(WalkParams P) {
  extern __shared__ __align__(16) unsigned char walk_raw[];   // WALK_WARPS x WalkSmem (dynamic)
  WalkSmem* smem = reinterpret_cast<WalkSmem*>(walk_raw);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * WALK_WARPS + wib;
  if (w >= P.nsel || (P.nsel_dev && w >= *P.nsel_dev)) return;
  WalkSmem& S = smem[wib];
  const int gid = P.sel ? P.sel[w] : w;
  const int4 grp = P.groups[gid];
  const int s = grp.y + lane;
  WalkState W;
  W.lane = lane;
  W.gz = grp.z;
  const float4 o4 = P.xh[grp.y];
  W.o = make_float3(o4.x, o4.y, o4.z);
  W.oL = make_float3(o4.x - P.g.L[0], o4.y - P.g.L[1], o4.z - P.g.L[2]);
  W.ri = -1.f;
  W.xi = W.yi = W.zi = 0.f;
  if (lane < 27)
    S.shf[lane] = make_float4(shift_of(lane % 3, P.g.L[0]), shift_of((lane / 3) % 3, P.g.L[1]),
                              shift_of(lane / 9, P.g.L[2]), 0.f);
  float ax = 0.f, ay = 0.f, az = 0.f;      // absolute target position (top-cell range)
  bool tg = false;
  if (lane < grp.z) {
    tg = P.tsel ? P.tsel[s] == P.tsel_val : P.tgt[s] != 0;
    if (tg) {
      const float4 p = P.xh[s];
      ax = p.x;
      ay = p.y;
      az = p.z;
      W.xi = p.x - W.o.x;
      W.yi = p.y - W.o.y;
      W.zi = p.z - W.o.z;
      W.ri = P.reach[s];
    }
  }
  if (!__any_sync(FULL_MASK, tg)) {            // no target in this group (e.g. a re-walk round)
    if (MODE != MODE_NB && lane == 0 && !P.check) P.len[gid] = 0;
    return;
  }
  // NB + solve: a target whose root lies beyond its new list is walked again right here
  // (up to SPH_INWALK_PASSES passes) instead of waiting for a host round
  HLane H;
  H.h = H.hbs = H.l = H.u = 0.f;
  H.ev = 0;
  H.st = HS_DONE;
  H.it = 0;
  int nb_tot = 0;
  for (int pass = 0;; ++pass) {
  W.lo = make_float3(warp_min_f(tg ? W.xi : INFINITY), warp_min_f(tg ? W.yi : INFINITY),
                     warp_min_f(tg ? W.zi : INFINITY));
  W.hi = make_float3(warp_max_f(tg ? W.xi : -INFINITY), warp_max_f(tg ? W.yi : -INFINITY),
                     warp_max_f(tg ? W.zi : -INFINITY));
  const float alo[3] = {warp_min_f(tg ? ax : INFINITY), warp_min_f(tg ? ay : INFINITY), warp_min_f(tg ? az : INFINITY)};
  const float ahi[3] = {warp_max_f(tg ? ax : -INFINITY), warp_max_f(tg ? ay : -INFINITY),
                        warp_max_f(tg ? az : -INFINITY)};
  W.R = warp_max_f(tg ? W.ri : 0.f);
  {
    // the targets' spheres, compacted, for the node tests; worth it only when the group's
    // reach is uneven or its targets are spread wider than their reach
    const unsigned tb = __ballot_sync(FULL_MASK, tg);
    W.ntg = __popc(tb);
    if (tg) {
      // stored in a stride-4 interleave of the (Morton-ordered) targets, so the first ones
      // tested span the group and a reached node usually meets a hit within the first vote
      const int pidx = __popc(tb & lanemask_lt()), q4 = (W.ntg + 3) >> 2;
      const int r4 = pidx & 3, c4 = pidx >> 2;
      const int full = W.ntg - 4 * (q4 - 1);   // rows 0..full-1 hold q4 entries, the rest q4 - 1
      const int slot = r4 < full ? r4 * q4 + c4 : full * q4 + (r4 - full) * (q4 - 1) + c4;
      S.tgt[slot] = make_float4(W.xi, W.yi, W.zi, reach_eff(W.ri, P.slack));
    }
    __syncwarp();
    const float rmin = warp_min_f(tg ? W.ri : INFINITY);
    const float dx = W.hi.x - W.lo.x, dy = W.hi.y - W.lo.y, dz = W.hi.z - W.lo.z;
    W.spheres = W.ntg <= 8 || rmin < 0.75f * W.R || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) > 0.25f * W.R * W.R;
  }
  W.cur = 0;
  W.raw = 0;
#ifdef SPH_WALK_STATS
  W.st_surv = 0;
  W.st_calls = 0;
#endif
#if NB_ROWS
  W.base = MODE == MODE_FILL ? P.off[gid] : (MODE == MODE_NB ? (int64_t)s * P.K : 0);
#else
  W.base = MODE == MODE_FILL ? P.off[gid] : (MODE == MODE_NB ? (int64_t)grp.y * P.K + lane : 0);
#endif
  if (MODE == MODE_NB && P.ovf && tg) W.base = P.ovf_off[s];
  int nq = 0;
  if (__any_sync(FULL_MASK, tg)) {
    // top cells (unwrapped indices) overlapping the box grown by the largest possible reach
    const float rmax = P.reach_max_bits ? __uint_as_float((unsigned)*P.reach_max_bits) : P.reach_max;
    const float Rw = reach_eff(MODE == MODE_NB ? W.R : fmaxf(W.R, rmax), P.slack) + P.slack;
    int a0[3], na[3];
    int T = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float E = P.g.E[0][a];
      int lo_i = (int)floorf((alo[a] - Rw) / E), hi_i = (int)floorf((ahi[a] + Rw) / E);
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
      if (ent != -1) {
        S.stk[__popc(sb & lanemask_lt())] = ent;
        if (MODE != MODE_NB) S.hint[__popc(sb & lanemask_lt())] = 0;
      }
      int top = __popc(sb);
      __syncwarp();
      while (top > 0) {
        int k = min(32, top);
        while (k > 0 && top - k + 8 * k > WALK_CAP) --k;
        if (k == 0) {                                  // frontier full: one subtree depth-first
          const int e = S.stk[top - 1];
          __syncwarp();
          --top;
          dfs_subtree<MODE>(P, W, S, S.stk + top, e, nq);
          continue;
        }
        int e = 0, hn = 0;
        if (lane < k) {
          e = S.stk[top - k + lane];
          if (MODE != MODE_NB) hn = S.hint[top - k + lane];
        }
        __syncwarp();
        top -= k;
        const int nd = e & SPH_IDX_MASK, code = (int)((unsigned)e >> SPH_IDX_BITS);
        bool reach = false, leaf = false, srt = false;
        int4 rec = make_int4(0, 0, -1, 0);
        if (lane < k) {
          rec = P.N.rec[nd];
          reach = node_in_reach<MODE>(P, W, S, nd, code);
        }
        int fh = 0;
        reach = node_in_spheres<MODE>(P, W, S, nd, code, reach, hn, &fh);
        if (lane < k) {
          leaf = reach && !(rec.z >= 0 && rec.y > WALK_TAKE);
          srt = leaf && P.any_sorted && P.N.sortoff[nd] >= 0;
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
        for (int c2 = 0; c2 < nch; ++c2) {
          S.stk[top + pre - nch + c2] = (rec.z + c2) | (code << SPH_IDX_BITS);
          if (MODE != MODE_NB) S.hint[top + pre - nch + c2] = (uint8_t)fh;
        }
        top += tot;
        // reached unsorted leaves: queue their ranges
        const bool ql = leaf && !srt;
        const unsigned qb = __ballot_sync(FULL_MASK, ql);
        if (nq + __popc(qb) > WALK_RQ) flush_ranges<MODE>(P, W, S, nq);
        if (qb) {
          const int q = nq + __popc(qb & lanemask_lt());
          if (ql) {
            S.rq_first[q] = rec.x;
            S.rq_code[q] = code;
            const int cx = code % 3, cy = (code / 3) % 3, cz = code / 9;
            S.rq_so[q] = make_float4(cx == 1 ? -P.g.L[0] : 0.f, cy == 1 ? -P.g.L[1] : 0.f, cz == 1 ? -P.g.L[2] : 0.f, 0.f);
            S.rq_oo[q] = make_float4(cx == 2 ? W.oL.x : W.o.x, cy == 2 ? W.oL.y : W.o.y, cz == 2 ? W.oL.z : W.o.z, 0.f);
          }
          // prefix of the new counts (one per queuing lane, in lane order)
          int v0 = ql ? rec.y : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL_MASK, v0, o);
            if (lane >= o) v0 += y;
          }
          const int basep = nq == 0 ? 0 : S.rq_pre[nq];
          __syncwarp();
          if (lane == 0 && nq == 0) S.rq_pre[0] = 0;
          if (ql) S.rq_pre[q + 1] = basep + v0;
          __syncwarp();
          nq += __popc(qb);
        }
        // reached sorted leaves: windowed sweeps, one at a time
        unsigned sbm = __ballot_sync(FULL_MASK, srt);
        while (sbm) {
          const int src = __ffs(sbm) - 1;
          sbm &= sbm - 1;
          const int snd = __shfl_sync(FULL_MASK, nd, src), scode = __shfl_sync(FULL_MASK, code, src);
          flush_ranges<MODE>(P, W, S, nq);
          sweep_node<MODE>(P, W, S, snd, scode);
        }
      }
    }
    flush_ranges<MODE>(P, W, S, nq);
  }
  if (lane == 0) {
    atomicAdd(&P.ctr[C_TMP2], (unsigned long long)W.raw);
    atomicMax(&P.ctr[C_TMP0], (unsigned long long)W.raw);
    if (P.raw_out) atomicAdd(P.raw_out, (unsigned long long)W.raw);
  }
#ifdef SPH_WALK_TRACE
  if (W.raw > 10000) {
    const int mc = __reduce_max_sync(FULL_MASK, tg ? W.cur : 0);
    if (lane == 0)
      printf("heavy walk mode %d group %d: targets %d R %.3g bbox %.3g %.3g %.3g spheres %d raw %d max list %d\n", MODE,
             gid, W.ntg, W.R, W.hi.x - W.lo.x, W.hi.y - W.lo.y, W.hi.z - W.lo.z, (int)W.spheres, W.raw, mc);
  }
#endif
#ifdef SPH_WALK_STATS
  if (MODE == MODE_NB && P.solve) {
    const int act = __popc(__ballot_sync(FULL_MASK, tg));
    const int rec = warp_sum_i(tg ? min(W.cur, P.K) : 0);
    if (lane == 0) {
      const int pp = min(pass, 7);
      atomicAdd(&g_walkstats[pp][0], 1ull);
      atomicAdd(&g_walkstats[pp][1], (unsigned long long)act);
      atomicAdd(&g_walkstats[pp][2], (unsigned long long)W.st_surv);
      atomicAdd(&g_walkstats[pp][3], (unsigned long long)rec);
      atomicAdd(&g_walkstats[pp][4], (unsigned long long)W.st_calls);
    }
  }
#endif
  if (MODE == MODE_NB && !P.ovf) nb_tot += tg ? min(W.cur, P.K) : 0;
  if (MODE == MODE_NB && P.solve) {
    // fused h iteration on the list just recorded (still in L1/L2): first overflow of K ->
    // shrink h_build; repeat overflow -> exact list in the pool (k_hsolve_pool)
    const int cnt = W.cur;
    bool act = tg;
    if (tg) {
      if (pass == 0) {
        H.h = P.xh[s].w;
        H.l = P.lo[s];
        H.u = P.hi[s];
      }
      H.hbs = W.ri;
      const bool over = cnt > P.K;
      if (over && P.shrunk[s]) {
        H.st = HS_OVF;
        act = false;
        P.ovf_cnt[s] = cnt;
      } else {
        if (over) P.shrunk[s] = 1;
        P.ovf_off_w[s] = -1;
        P.ovf_cnt[s] = 0;
      }
    }
#if NB_PREFETCH
    if (act && NB_ROWS) {   // pull the row's lines into L1 at once (the sums then hit L1)
      const char* rb = reinterpret_cast<const char*>(P.nb_r2 + (int64_t)s * P.K);
      const int bytes = min(cnt, P.K) * 4;
      for (int b = 0; b < bytes; b += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(rb + b));
    }
#endif
    __syncwarp();   // the lists recorded by every lane are visible to the cooperative sums
    warp_hsolve(act, P.nb_r2 + (NB_ROWS ? (int64_t)s * P.K : (int64_t)grp.y * P.K + lane), NB_ROWS ? 1 : W.gz, cnt, P.K,
                false, true, H, P.n_t, P.tol, P.margin,
                P.hcap, P.max_iter);
    if (tg) {
      reinterpret_cast<float*>(const_cast<float4*>(P.xh) + s)[3] = H.h;
      P.hb_w[s] = H.hbs;
      P.lo[s] = H.l;
      P.hi[s] = H.u;
      P.state[s] = H.st;
      P.nb_cnt[s] = cnt;
    }
    const bool again = tg && H.st == HS_REGROW && pass + 1 < SPH_INWALK_PASSES;
    // lanes that finish in this pass (converged, unconverged, overflowed, or out of passes)
    // are counted now; the re-walked ones in the pass that finishes them
    hsolve_count(tg && !again, H, P.hc);
    if (__any_sync(FULL_MASK, again)) {
      tg = again;
      W.ri = again ? H.hbs : -1.f;
      continue;
    }
    if (P.rg_out) {
      const unsigned rg = __ballot_sync(FULL_MASK, tg && H.st == HS_REGROW);
      if (rg && lane == 0) P.rg_out[atomicAdd(P.rg_cnt, 1)] = gid;
    }
  }
  break;
  }   // passes
  if (MODE == MODE_NB) {
    if (tg && !P.ovf && !P.solve) P.nb_cnt[s] = W.cur;
    if (!P.ovf && P.nb_entries) {
      const int tot = warp_sum_i(nb_tot);
      if (lane == 0 && tot) atomicAdd(P.nb_entries, (unsigned long long)tot);
    } else if (P.ovf && P.nb_entries) {
      const int tot = warp_sum_i(tg ? W.cur : 0);
      if (lane == 0 && tot) atomicAdd(P.nb_entries, (unsigned long long)tot);
    }
  } else if (MODE == MODE_COUNT) {
    if (lane == 0) {
      P.len[gid] = W.cur;
      if (P.len_sel) P.len_sel[w] = W.cur;
    }
  } else if (lane == 0) {
    if (!P.check) P.len[gid] = W.cur;
    else if (W.cur != P.len[gid]) atomicOr(&P.ctr[C_ERR], 1ull << 20);   // pass mismatch
  }
}

// list offsets of the selected groups: base + exclusive scan of their lengths
__global__ void k_set_offsets(int nsel, const int* __restrict__ sel, const int64_t* __restrict__ scan, int64_t base,
                              int64_t* __restrict__ off) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nsel) return;
  off[sel ? sel[w] : w] = base + scan[w];
}

__global__ void k_compact_idx(const int* __restrict__ flag, const int* __restrict__ scan, int64_t n,
                              int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[scan[i]] = (int32_t)i;
}
__global__ void k_ovf_offsets(int64_t n, const int64_t* __restrict__ c, const int64_t* __restrict__ scan,
                              int64_t base, int64_t* __restrict__ off) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    if (c[s] > 0) off[s] = base + scan[s];
}

// groups whose UNION list exceeded the slab capacity: compaction flags and their lengths
__global__ void k_union_overflow(int ng, const int* __restrict__ len, int cap, int* __restrict__ flag) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < ng) flag[g] = len[g] > cap ? 1 : 0;
}
__global__ void k_gather_len(int nsel, const int* __restrict__ sel, const int* __restrict__ len,
                             int64_t* __restrict__ out) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < nsel) out[w] = len[sel[w]];
}
__global__ void k_slab_offsets(int ng, int cap, int64_t* __restrict__ off) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < ng) off[g] = (int64_t)g * cap;
}

__global__ void k_flag_pos64(const int64_t* __restrict__ c, int64_t n, int* __restrict__ flag) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    flag[s] = c[s] > 0 ? 1 : 0;
}
__global__ void k_compact_append(const int* __restrict__ flag, const int* __restrict__ scan, int64_t n,
                                 int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[scan[i]] = (int32_t)i;
}
