// interact.cuh — density and force loops over the cell hierarchy with sorted pair sweeps.
//
// Work unit: one warp per (leaf cell, chunk of 32 particles); lane = target particle i.
// A warp visits, in a fixed order,
//   * the leaf's self interaction (all particles of the leaf), then
//   * for the leaf and each ancestor, every KEPT pair slot (cell Y at offset k): the
//     sorted sweep of P:644-669 along canonical direction d = dir(k). Y's particles are
//     traversed in ascending key order when Y lies on the +d side and descending when it
//     lies on the -d side (the "flip" of P:693-698), and the sweep stops at the first
//     source whose projected distance exceeds every lane's window (the early exit of
//     P:653/P:663). Sources are staged 32 at a time in shared memory with float4 loads;
//     each lane then tests them against its own target (gather form: the j-side update
//     of the paper's pair task is the i-side of the mirrored slot, so no atomics).
// Density window = h_i (r < h_i, Eq. 2); force window = max(h_i, max h in Y)
// (r < max(h_i, h_j), Eq. 4).
#pragma once
#include "build.cuh"

// per-particle h-iteration state
#define HS_DONE 0
#define HS_ACTIVE 1
#define HS_PARKED 2   // wants h beyond the top cells: waits for a rebuild
#define HS_COARSE 3   // h beyond its cells' h_build: evaluated over the 27 top cells (coarse_gather)

struct TravParams {
  const uint8_t* tau;       // interaction level per particle (cell order)
  const int4* tasks;        // {leaf cell, first particle (cell order), count <= 32, -}
  int ntasks;
  NodeArrays N;
  LevelGeom g;
  const SortEntry* sorted;
  const SegDesc* seg;       // per (cell, kind) source-list descriptors
  const int* segoff2;
  const int* segcnt2;
  const uint8_t* active;   // null = all
  float slack;             // absolute window slack (fp32 rounding of keys/corners)
  int dbg_skip;             // debug only: bit k skips kind k (wrong results; timing experiments)
  int desc_min;             // culling descends into cells holding more particles than this
  unsigned long long* ctr;
};

// ------------------------------------------------------------------ density ------
struct DensOp {
  struct Src {
    float4 a;  // x, y, z (shifted), unused
    float4 b;  // vx, vy, vz, m
  };
  const float4* __restrict__ xh;
  const float4* __restrict__ vm;
  bool valid, act;
  bool nonly;        // N(h) and its derivatives only (a pass that cannot converge anyone)
  int s;
  float x0, y0, z0;  // unshifted target position
  float xi, yi, zi;  // shifted for the current segment
  float hi, hi2, hinv, vxi, vyi, vzi;
  double sf;
  float smf, smqfp, sqfp, divs, crx, cry, crz;
  float sq2fpp;        // sum q^2 f''(q): second derivative of N(h) for the Halley step
  int cnt;
  long long ncand, nself, nseg, nchunk;

  __device__ __forceinline__ void init(int s_, bool v) {
    s = s_;
    valid = v;
    nself = nseg = nchunk = 0;
    sf = 0.0;
    smf = smqfp = sqfp = divs = crx = cry = crz = 0.f;
    sq2fpp = 0.f;
    cnt = 0;
    ncand = 0;
    if (v) {
      float4 p = xh[s];
      float4 q = vm[s];
      x0 = p.x; y0 = p.y; z0 = p.z;
      hi = p.w;
      vxi = q.x; vyi = q.y; vzi = q.z;
    } else {
      x0 = y0 = z0 = 0.f;
      hi = 0.f;
      vxi = vyi = vzi = 0.f;
    }
    hi2 = hi * hi;
    hinv = v ? 1.0f / hi : 0.f;
    xi = x0; yi = y0; zi = z0;
  }
  __device__ __forceinline__ float window(float) const { return hi; }
  __device__ __forceinline__ void shift(float tx, float ty, float tz) {
    xi = x0 + tx; yi = y0 + ty; zi = z0 + tz;
  }
  __device__ __forceinline__ void stage(Src& d, int j, float sx, float sy, float sz) const {
    float4 p = xh[j];
    d.a = make_float4(p.x + sx, p.y + sy, p.z + sz, 0.f);
    d.b = vm[j];
  }
  // box filter support: reach of a source list, and the fields staged for survivors
  static constexpr bool kListHmax = false;
  __device__ __forceinline__ float reach(float hmt, float) const { return hmt; }
  __device__ __forceinline__ float target_reach() const { return hi; }
  __device__ __forceinline__ float4 src_pos(int j) const { return xh[j]; }
  __device__ __forceinline__ void stage_rest(Src& d, int j, float4 ps) const {
    d.a = make_float4(ps.x, ps.y, ps.z, 0.f);
    if (!nonly) d.b = vm[j];
  }
  __device__ __forceinline__ bool test(const Src& src) const {
    const float dx = xi - src.a.x, dy = yi - src.a.y, dz = zi - src.a.z;
    return fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < hi2;
  }
  __device__ __forceinline__ void interact(const Src& src, bool is_self) {
    const float dx = xi - src.a.x, dy = yi - src.a.y, dz = zi - src.a.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    if (r2 < hi2) {
      const float rinv = r2 > 0.f ? rsqrtf(r2) : 0.f;
      const float r = r2 * rinv;
      const float q = r * hinv;
      float f, fp, fpp;
      if (q <= 0.5f) {
        f = fmaf(q * q, fmaf(6.f, q, -6.f), 1.f);
        fp = q * fmaf(18.f, q, -12.f);
        fpp = fmaf(36.f, q, -12.f);
      } else {
        const float t = 1.f - q;
        f = 2.f * t * t * t;
        fp = -6.f * t * t;
        fpp = 12.f * t;
      }
      sf += (double)f;
      sq2fpp = fmaf(q * q, fpp, sq2fpp);
      const float qfp = q * fp;
      sqfp += qfp;
      if (nonly) return;
      const float mj = src.b.w;
      smf = fmaf(mj, f, smf);
      smqfp = fmaf(mj, qfp, smqfp);
      const float gf = mj * fp * rinv;
      const float dvx = src.b.x - vxi, dvy = src.b.y - vyi, dvz = src.b.z - vzi;
      divs = fmaf(gf, fmaf(dvx, dx, fmaf(dvy, dy, dvz * dz)), divs);
      crx = fmaf(gf, dvy * dz - dvz * dy, crx);
      cry = fmaf(gf, dvz * dx - dvx * dz, cry);
      crz = fmaf(gf, dvx * dy - dvy * dx, crz);
      cnt += is_self ? 0 : 1;
    }
  }
};

// ------------------------------------------------------------------ force --------
struct ForceOp {
  struct Src {
    float4 a;  // x, y, z (shifted), 1/h
    float4 b;  // vx, vy, vz, m
    float4 c;  // A~ = A * (8/pi) h^-4, rho, c, f
  };
  const float4* __restrict__ fx;
  const float4* __restrict__ vm;
  const float4* __restrict__ fs;
  float alpha;
  bool valid, act;
  int s;
  float x0, y0, z0, xi, yi, zi;
  float hi, hi2, hinv, hhat, At, rhoi, ci, fi, vxi, vyi, vzi;
  float ax, ay, az, du, vsig;
  int cnt;
  long long ncand, nself, nseg, nchunk;

  __device__ __forceinline__ void init(int s_, bool v) {
    s = s_;
    valid = v;
    nself = nseg = nchunk = 0;
    ax = ay = az = du = vsig = 0.f;
    cnt = 0;
    ncand = 0;
    if (v) {
      float4 p = fx[s], q = vm[s], w = fs[s];
      x0 = p.x; y0 = p.y; z0 = p.z;
      hinv = p.w;
      hi = 1.0f / hinv;
      vxi = q.x; vyi = q.y; vzi = q.z;
      At = w.x; rhoi = w.y; ci = w.z; fi = w.w;
    } else {
      x0 = y0 = z0 = 0.f;
      hinv = 0.f; hi = 0.f;
      vxi = vyi = vzi = 0.f;
      At = rhoi = ci = fi = 0.f;
    }
    hi2 = hi * hi;
    const float h2i = hinv * hinv;
    hhat = SPH_CNORM * h2i * h2i;
    xi = x0; yi = y0; zi = z0;
  }
  __device__ __forceinline__ float window(float hmax_list) const { return fmaxf(hi, hmax_list); }
  __device__ __forceinline__ void shift(float tx, float ty, float tz) {
    xi = x0 + tx; yi = y0 + ty; zi = z0 + tz;
  }
  __device__ __forceinline__ void stage(Src& d, int j, float sx, float sy, float sz) const {
    float4 p = fx[j];
    d.a = make_float4(p.x + sx, p.y + sy, p.z + sz, p.w);
    d.b = vm[j];
    d.c = fs[j];
  }
  static constexpr bool kListHmax = true;
  __device__ __forceinline__ float reach(float hmt, float hmax_list) const { return fmaxf(hmt, hmax_list); }
  __device__ __forceinline__ float target_reach() const { return hi; }
  __device__ __forceinline__ float4 src_pos(int j) const { return fx[j]; }
  __device__ __forceinline__ void stage_rest(Src& d, int j, float4 ps) const {
    d.a = ps;
    d.b = vm[j];
    d.c = fs[j];
  }
  __device__ __forceinline__ static float fprime(float q) {
    if (q <= 0.5f) return q * fmaf(18.f, q, -12.f);
    const float t = 1.f - q;
    return -6.f * t * t;
  }
  __device__ __forceinline__ bool test(const Src& src) const {
    const float dx = xi - src.a.x, dy = yi - src.a.y, dz = zi - src.a.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    return r2 < hi2 || r2 * (src.a.w * src.a.w) < 1.0f;
  }
  __device__ __forceinline__ void interact(const Src& src, bool is_self) {
    const float dx = xi - src.a.x, dy = yi - src.a.y, dz = zi - src.a.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float hjinv = src.a.w;
    const float hj2i = hjinv * hjinv;
    const bool in_i = r2 < hi2;
    const bool in_j = r2 * hj2i < 1.0f;
    if ((in_i || in_j) && !is_self) {
      const float rinv = r2 > 0.f ? rsqrtf(r2) : 0.f;
      const float r = r2 * rinv;
      const float fpi = in_i ? fprime(r * hinv) : 0.f;
      const float fpj = in_j ? fprime(r * hjinv) : 0.f;
      const float hhatj = SPH_CNORM * hj2i * hj2i;
      const float Gi = hhat * fpi * rinv;
      const float Gj = hhatj * fpj * rinv;
      const float vx = vxi - src.b.x, vy = vyi - src.b.y, vz = vzi - src.b.z;
      const float vdx = fmaf(vx, dx, fmaf(vy, dy, vz * dz));
      const float w = fminf(0.f, vdx * rinv);
      const float cs = ci + src.c.z - 3.f * w;
      const float Pi = -alpha * cs * w / (rhoi + src.c.y);
      const float V = Pi * (fi + src.c.w) * (Gi + Gj);
      const float AGi = At * fpi * rinv;
      const float AGj = src.c.x * fpj * rinv;
      const float T = AGi + AGj + 0.25f * V;
      const float mj = src.b.w;
      const float mT = mj * T;
      ax = fmaf(-mT, dx, ax);
      ay = fmaf(-mT, dy, ay);
      az = fmaf(-mT, dz, az);
      du = fmaf(mj * vdx, AGi + 0.125f * V, du);
      vsig = fmaxf(vsig, cs);
      cnt += 1;
    }
  }
};

// ------------------------------------------------------------------ traversal ----
struct WarpBox {
  float3 lo, hi;  // bounding box of the warp's participating targets (unshifted)
  float hmax;     // max target window base (h_i)
};

template <class Op>
__device__ __forceinline__ WarpBox warp_box(const Op& op) {
  WarpBox b;
  b.lo = make_float3(warp_min_f(op.act ? op.x0 : INFINITY), warp_min_f(op.act ? op.y0 : INFINITY),
                     warp_min_f(op.act ? op.z0 : INFINITY));
  b.hi = make_float3(warp_max_f(op.act ? op.x0 : -INFINITY), warp_max_f(op.act ? op.y0 : -INFINITY),
                     warp_max_f(op.act ? op.z0 : -INFINITY));
  b.hmax = warp_max_f(op.act ? op.target_reach() : 0.f);
  return b;
}

// One source list swept by the warp. windowed: sorted sweep with early exit at the first
// entry beyond every lane's window (Lw = warp-wide limit on the key); otherwise the whole
// list. Each chunk of 32 entries (keys, indices and positions read coalesced) is filtered
// by a sphere/box test against the participating targets' bounding box (reach = max target
// window, or the list's max h for the force); survivors are staged in shared memory and
// every participating lane tests them.
template <class Op>
__device__ __forceinline__ void seg_list(Op& op, const TravParams& P, const WarpBox& B, int64_t off, int cnt,
                                         bool windowed, bool range, bool flip, float Lw, float sox, float soy,
                                         float soz, float tox, float toy, float toz, float reach, bool selfcheck,
                                         typename Op::Src* sm, int* smj, int lane) {
  const SortEntry* __restrict__ list = P.sorted + off;
  const float blx = B.lo.x + tox, bly = B.lo.y + toy, blz = B.lo.z + toz;
  const float bhx = B.hi.x + tox, bhy = B.hi.y + toy, bhz = B.hi.z + toz;
  const float rr = fmaf(reach, 1.00001f, P.slack);
  const float rr2 = rr * rr;
  op.nseg += 1;
  for (int base = 0; base < cnt; base += 32) {
    op.nchunk += 1;
    const int e = base + lane;
    bool in = false, keep = false;
    int j = 0;
    float4 ps;
    if (e < cnt) {
      if (range) {                       // the cell's own contiguous range (cell order)
        j = (int)off + e;
        in = true;
      } else {
        const int ei = flip ? cnt - 1 - e : e;
        const SortEntry en = list[ei];
        in = !windowed || (flip ? (en.key > Lw) : (en.key < Lw));
        j = en.idx;
      }
      const float4 pr = op.src_pos(j);
      ps = make_float4(pr.x + sox, pr.y + soy, pr.z + soz, pr.w);
      const float ex = fmaxf(fmaxf(blx - ps.x, ps.x - bhx), 0.f);
      const float ey = fmaxf(fmaxf(bly - ps.y, ps.y - bhy), 0.f);
      const float ez = fmaxf(fmaxf(blz - ps.z, ps.z - bhz), 0.f);
      keep = in && fmaf(ex, ex, fmaf(ey, ey, ez * ez)) < rr2;
    }
    const unsigned bal_in = __ballot_sync(FULL_MASK, in);
    const unsigned bal = __ballot_sync(FULL_MASK, keep);
    const int m = __popc(bal);
    if (keep) {
      const int pos = __popc(bal & lanemask_lt());
      op.stage_rest(sm[pos], j, ps);
      smj[pos] = j;
    }
    __syncwarp();
    if (op.act && !(P.dbg_skip & 4)) {
      // two phases: distance tests of all staged sources into a hit mask, then the
      // interaction body only for the hits (a lane's misses cost no body instructions)
      op.ncand += m;
      unsigned hm = 0u;
#pragma unroll 4
      for (int t = 0; t < m; ++t) hm |= (unsigned)op.test(sm[t]) << t;
      while (hm) {
        const int t = __ffs(hm) - 1;
        hm &= hm - 1;
        op.interact(sm[t], selfcheck && smj[t] == op.s);
      }
    }
    __syncwarp();
    if (__popc(bal_in) < 32) break;
  }
}

// Whole-cell ranges swept as one flattened stream: the sub-cell ranges collected by the
// culling descent (cull_range) are streamed in chunks of 32 without per-range set-up.
#define RBUF 64
struct WarpSmemT {
  SegDesc sd[27];
  int rs[RBUF];        // range starts (cell order)
  int rc[RBUF + 1];    // exclusive prefix of range counts
  int rcode[RBUF];     // target shift code (bits 0-2) | self check (bit 3) | source shift (bits 4-6) |
                       // tau filter (bit 7, keep tau >= bits 8-11)
  float rreach[RBUF];  // reach of the range's list (force: includes the list's max h)
  int stk[96];
  int nr;
};

template <class Op>
__device__ __forceinline__ void flush_ranges(Op& op, const TravParams& P, const WarpBox& B, WarpSmemT& W, float reach,
                                             typename Op::Src* sm, int* smj, int* smc, int lane) {
  const int nr = W.nr;
  if (nr == 0) return;
  // exclusive prefix of the (<= 64) range counts
  int c0 = lane < nr ? W.rc[lane] : 0, c1 = lane + 32 < nr ? W.rc[lane + 32] : 0;
  int i0 = c0, i1 = c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y0 = __shfl_up_sync(FULL_MASK, i0, o), y1 = __shfl_up_sync(FULL_MASK, i1, o);
    if (lane >= o) { i0 += y0; i1 += y1; }
  }
  const int t0 = __shfl_sync(FULL_MASK, i0, 31);
  __syncwarp();
  if (lane < nr) W.rc[lane] = i0 - c0;
  if (lane + 32 < nr) W.rc[lane + 32] = t0 + i1 - c1;
  const int total = t0 + __shfl_sync(FULL_MASK, i1, 31);
  if (lane == 0) W.rc[nr] = total;
  __syncwarp();
  (void)reach;
  op.nseg += 1;
  for (int base = 0; base < total; base += 32) {
    op.nchunk += 1;
    const int g = base + lane;
    bool keep = false;
    int j = 0, code = 0;
    float4 ps;
    if (g < total) {
      int t = 0;                               // range of entry g: rc[t] <= g < rc[t+1]
#pragma unroll
      for (int step = 32; step > 0; step >>= 1)
        if (t + step < nr && W.rc[t + step] <= g) t += step;
      j = W.rs[t] + (g - W.rc[t]);
      code = W.rcode[t];
      const float rrt = fmaf(W.rreach[t], 1.00001f, P.slack);
      const float sox = (code & 16) ? -P.g.L[0] : 0.f, soy = (code & 32) ? -P.g.L[1] : 0.f,
                  soz = (code & 64) ? -P.g.L[2] : 0.f;
      const float tox = (code & 1) ? -P.g.L[0] : 0.f, toy = (code & 2) ? -P.g.L[1] : 0.f,
                  toz = (code & 4) ? -P.g.L[2] : 0.f;
      const float4 pr = op.src_pos(j);
      ps = make_float4(pr.x + sox, pr.y + soy, pr.z + soz, pr.w);
      const float ex = fmaxf(fmaxf(B.lo.x + tox - ps.x, ps.x - (B.hi.x + tox)), 0.f);
      const float ey = fmaxf(fmaxf(B.lo.y + toy - ps.y, ps.y - (B.hi.y + toy)), 0.f);
      const float ez = fmaxf(fmaxf(B.lo.z + toz - ps.z, ps.z - (B.hi.z + toz)), 0.f);
      keep = fmaf(ex, ex, fmaf(ey, ey, ez * ez)) < rrt * rrt;
      if (keep && (code & 128)) keep = (int)P.tau[j] >= ((code >> 8) & 15);   // list A membership
    }
    const unsigned bal = __ballot_sync(FULL_MASK, keep);
    const int m = __popc(bal);
    if (keep) {
      const int pos = __popc(bal & lanemask_lt());
      op.stage_rest(sm[pos], j, ps);
      smj[pos] = j;
      smc[pos] = code;
    }
    __syncwarp();
    if (op.act && !(P.dbg_skip & 4)) {
      op.ncand += m;
      unsigned hm = 0u;
      for (int t = 0; t < m; ++t) {
        const int cd = smc[t];
        bool hit;
        if (cd & 7) {                          // periodic image: shift the target (exact side)
          op.shift((cd & 1) ? -P.g.L[0] : 0.f, (cd & 2) ? -P.g.L[1] : 0.f, (cd & 4) ? -P.g.L[2] : 0.f);
          hit = op.test(sm[t]);
          op.shift(0.f, 0.f, 0.f);
        } else {
          hit = op.test(sm[t]);
        }
        hm |= (unsigned)hit << t;
      }
      while (hm) {
        const int t = __ffs(hm) - 1;
        hm &= hm - 1;
        const int cd = smc[t];
        if (cd & 7) {
          op.shift((cd & 1) ? -P.g.L[0] : 0.f, (cd & 2) ? -P.g.L[1] : 0.f, (cd & 4) ? -P.g.L[2] : 0.f);
          op.interact(sm[t], false);
          op.shift(0.f, 0.f, 0.f);
        } else {
          op.interact(sm[t], (cd & 8) && smj[t] == op.s);
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) W.nr = 0;
  __syncwarp();
}

// distance from the target box (shifted by the target shift) to a cell box
__device__ __forceinline__ float box_gap2(const WarpBox& B, float tox, float toy, float toz, float cx, float cy,
                                          float cz, float ex, float ey, float ez) {
  const float gx = fmaxf(fmaxf(cx - (B.hi.x + tox), (B.lo.x + tox) - (cx + ex)), 0.f);
  const float gy = fmaxf(fmaxf(cy - (B.hi.y + toy), (B.lo.y + toy) - (cy + ey)), 0.f);
  const float gz = fmaxf(fmaxf(cz - (B.hi.z + toz), (B.lo.z + toz) - (cz + ez)), 0.f);
  return fmaf(gx, gx, fmaf(gy, gy, gz * gz));
}

// A neighbour cell whose list is its whole particle range: descend into its sub-cells and
// collect (into the range buffer) only those within reach of the targets' box. The cell's
// range in cell (Morton) order is the concatenation of its children's ranges.
template <class Op>
__device__ __forceinline__ void cull_range(Op& op, const TravParams& P, const WarpBox& B, WarpSmemT& W,
                                           const SegDesc& d, int level, float reach, bool kindA,
                                           typename Op::Src* sm, int* smj, int* smc, int lane) {
  const int tf = (d.meta & (1 << 15)) ? (128 | (level << 8)) : 0;
  const int cx = (d.meta >> 8) & 3, cy = (d.meta >> 10) & 3, cz = (d.meta >> 12) & 3;
  const float tox = cx == 1 ? -P.g.L[0] : 0.f, toy = cy == 1 ? -P.g.L[1] : 0.f, toz = cz == 1 ? -P.g.L[2] : 0.f;
  const float sox = cx == 2 ? -P.g.L[0] : 0.f, soy = cy == 2 ? -P.g.L[1] : 0.f, soz = cz == 2 ? -P.g.L[2] : 0.f;
  const int code = (cx == 1 ? 1 : 0) | (cy == 1 ? 2 : 0) | (cz == 1 ? 4 : 0) | ((kindA && (d.meta & 64)) ? 8 : 0) |
                   (cx == 2 ? 16 : 0) | (cy == 2 ? 32 : 0) | (cz == 2 ? 64 : 0) | tf;
  const float rr = fmaf(reach, 1.00001f, P.slack);
  const float rr2 = rr * rr;
  int top = 0;
  if (lane == 0) W.stk[0] = d.Y;
  top = 1;
  __syncwarp();
  while (top > 0) {
    const int node = W.stk[--top];
    __syncwarp();
    const int cnt = P.N.count[node];
    const int4 ijk = P.N.ijk[node];
    int ch = -1;
    bool ok = false;
    if (cnt > P.desc_min && ijk.w < P.g.depth && lane < 8) {
      ch = P.N.child[8 * (int64_t)node + lane];
      if (ch >= 0) {
        const int4 cc = P.N.ijk[ch];
        const int l = cc.w;
        ok = box_gap2(B, tox, toy, toz, node_corner(cc.x, l, 0, P.g) + sox, node_corner(cc.y, l, 1, P.g) + soy,
                      node_corner(cc.z, l, 2, P.g) + soz, P.g.E[l][0], P.g.E[l][1], P.g.E[l][2]) < rr2;
      }
    }
    const unsigned anych = __ballot_sync(FULL_MASK, ch >= 0);
    if (anych == 0u) {                         // leaf (or small cell): take its whole range
      if (lane == 0) {
        W.rs[W.nr] = P.N.first[node];
        W.rc[W.nr] = cnt;
        W.rcode[W.nr] = code;
        W.rreach[W.nr] = reach;
        W.nr = W.nr + 1;
      }
      __syncwarp();
      if (W.nr == RBUF) flush_ranges(op, P, B, W, 0.f, sm, smj, smc, lane);
      continue;
    }
    const unsigned okb = __ballot_sync(FULL_MASK, ok);
    if (ok) W.stk[top + __popc(okb & lanemask_lt())] = ch;
    top += __popc(okb);
    __syncwarp();
  }
}

// The sources of one (cell X, kind) for the warp's targets: lists that are a cell's whole
// range are culled down its sub-cells and streamed together; presorted lists are swept with
// the windowed early exit; compacted lists are swept whole.
template <class Op>
__device__ __forceinline__ void sweep_cell(Op& op, const TravParams& P, const WarpBox& B, int X, int level, int kind,
                                           typename Op::Src* sm, int* smj, int* smc, WarpSmemT& W, int lane) {
  const int s0 = P.segoff2[2 * X + kind], ns = P.segcnt2[2 * X + kind];
  SegDesc mine;
  if (lane < ns) {
    mine = P.seg[s0 + lane];
    W.sd[lane] = mine;
  }
  __syncwarp();
  bool isrange = false;
  if (lane < ns) isrange = (mine.meta & (1 << 14)) != 0;
  const unsigned rb = __ballot_sync(FULL_MASK, isrange);
  const unsigned ob = __ballot_sync(FULL_MASK, lane < ns && !isrange);
  if (rb) {
    unsigned rem = rb;
#pragma unroll 1
    while (rem) {
      const int t = __ffs(rem) - 1;
      rem &= rem - 1;
      const float hl = Op::kListHmax ? (kind ? P.N.hmaxR[W.sd[t].Y] : P.N.hmaxA[W.sd[t].Y]) : 0.f;
      cull_range(op, P, B, W, W.sd[t], level, op.reach(B.hmax, hl), kind == 0, sm, smj, smc, lane);
    }
    flush_ranges(op, P, B, W, 0.f, sm, smj, smc, lane);
  }
  unsigned rem = ob;
#pragma unroll 1
  while (rem) {
    const int t = __ffs(rem) - 1;
    rem &= rem - 1;
    const SegDesc d = W.sd[t];
    const float hl = Op::kListHmax ? (kind ? P.N.hmaxR[d.Y] : P.N.hmaxA[d.Y]) : 0.f;
    const float reach = op.reach(B.hmax, hl);
    const int cx = (d.meta >> 8) & 3, cy = (d.meta >> 10) & 3, cz = (d.meta >> 12) & 3;
    // exact fp32 shifts: always subtract L from the copy that lies near L (Sterbenz)
    const float tox = cx == 1 ? -P.g.L[0] : 0.f, toy = cy == 1 ? -P.g.L[1] : 0.f, toz = cz == 1 ? -P.g.L[2] : 0.f;
    const float sox = cx == 2 ? -P.g.L[0] : 0.f, soy = cy == 2 ? -P.g.L[1] : 0.f, soz = cz == 2 ? -P.g.L[2] : 0.f;
    op.shift(tox, toy, toz);
    if (d.meta & 128) {                        // compacted list, swept whole
      seg_list(op, P, B, d.off, d.cnt, false, false, false, 0.f, sox, soy, soz, tox, toy, toz, reach,
               kind == 0 && (d.meta & 64), sm, smj, lane);
      continue;
    }
    const bool flip = (d.meta & 32) != 0;
    const float3 du = dir_unit(d.meta >> 16);
    const float pi = proj(op.xi - d.cx, op.yi - d.cy, op.zi - d.cz, du);   // target key in Y's frame
    const float wq = fmaf(op.window(hl), 1.00001f, P.slack);
    float lim = flip ? pi - wq : pi + wq;
    if (!op.act) lim = flip ? INFINITY : -INFINITY;
    const float Lw = flip ? warp_min_f(lim) : warp_max_f(lim);
    seg_list(op, P, B, d.off, d.cnt, true, false, flip, Lw, sox, soy, soz, tox, toy, toz, reach, false, sm, smj, lane);
  }
  op.shift(0.f, 0.f, 0.f);
  __syncwarp();
}

// Coarse gather for density targets whose h exceeds the h their cells were built for (state
// HS_COARSE): every partner within the top cell edge lies in the 27 top cells around the
// target, so their whole ranges, culled down to the targets' reach, give the one-sided sum
// of Eq. 2 exactly (no tau filter: each particle appears in exactly one top cell).
template <class Op>
__device__ __forceinline__ void coarse_gather(Op& op, const TravParams& P, int leaf, typename Op::Src* sm, int* smj,
                                              int* smc, WarpSmemT& W, int lane) {
  int X = leaf;
  while (P.N.parent[X] >= 0) X = P.N.parent[X];
  const WarpBox B = warp_box(op);
  const int4 cX = P.N.ijk[X];
  if (lane < 27) {
    const int k = lane;
    const int Y = (k == 13) ? X : P.N.slot[27 * (int64_t)X + k];
    SegDesc d;
    d.Y = Y;
    d.off = 0;
    d.cnt = 0;
    d.cx = d.cy = d.cz = 0.f;
    int meta = k | (1 << 14) | (k == 13 ? 64 : 0);
    if (Y >= 0 && k != 13) {
      const int4 cY = P.N.ijk[Y];
      const int dd[3] = {cX.x + off_x(k) - cY.x, cX.y + off_y(k) - cY.y, cX.z + off_z(k) - cY.z};
      for (int a = 0; a < 3; ++a) {
        const int sa = dd[a] > 1 ? 1 : (dd[a] < -1 ? -1 : 0);
        meta |= (sa > 0 ? 1 : (sa < 0 ? 2 : 0)) << (8 + 2 * a);
      }
    }
    d.meta = meta;
    W.sd[lane] = d;
  }
  __syncwarp();
#pragma unroll 1
  for (int k = 0; k < 27; ++k) {
    if (W.sd[k].Y < 0) continue;
    cull_range(op, P, B, W, W.sd[k], 0, op.reach(B.hmax, 0.f), true, sm, smj, smc, lane);
  }
  flush_ranges(op, P, B, W, 0.f, sm, smj, smc, lane);
}

// Visit every pair of the warp's targets exactly once:
// at each level l of the leaf's ancestor chain, targets with tau == l sweep list A of the
// 27 cells around their level-l cell, targets with tau > l sweep list R (the partners with
// tau_j == l < tau_i, enumerated at min(tau_i, tau_j)).
template <class Op>
__device__ __forceinline__ void traverse(Op& op, const TravParams& P, int leaf, typename Op::Src* sm, int* smj,
                                         int* smc, WarpSmemT& W, int lane) {
  const int ti = op.valid ? (int)P.tau[op.s] : -1;
  const int tmax = (int)__reduce_max_sync(FULL_MASK, (unsigned)(ti + 1)) - 1;
  if (lane == 0) W.nr = 0;
  __syncwarp();
  int X = leaf;
  int level = P.N.ijk[leaf].w;
  while (X >= 0) {
    if (level <= tmax) {
#pragma unroll 1
      for (int kind = 1; kind >= 0; --kind) {   // R (deeper targets), then A (tau == l)
        op.act = op.valid && (kind ? ti > level : ti == level);
        if (!__any_sync(FULL_MASK, op.act)) continue;
        if (P.dbg_skip & (1 << kind)) continue;   // timing experiments only (SPH_DEBUG_SKIP)
        const WarpBox B = warp_box(op);
        sweep_cell(op, P, B, X, level, kind, sm, smj, smc, W, lane);
      }
    }
    X = P.N.parent[X];
    --level;
  }
}

#define INTERACT_WARPS 4
#ifndef SPH_DENS_MINB
#define SPH_DENS_MINB 6
#endif
#ifndef SPH_FORCE_MINB
#define SPH_FORCE_MINB 5
#endif

struct DensOut {
  int nonly;      // 1: N-only pass (k_h_update keeps every particle active)
  double* sf;
  float4* acc0;   // smf, smqfp, sqfp, divs
  float4* acc1;   // curl sums xyz, count (int bits)
  float* s2;      // sum q^2 f''(q)
};

__global__ void __launch_bounds__(INTERACT_WARPS * 32, SPH_DENS_MINB) k_density(TravParams P, const float4* __restrict__ xh,
                                                                 const float4* __restrict__ vm,
                                                                 const uint8_t* __restrict__ tau, DensOut out) {
  __shared__ DensOp::Src smem[INTERACT_WARPS][32];
  __shared__ int smj[INTERACT_WARPS][32];
  __shared__ int smc[INTERACT_WARPS][32];
  __shared__ WarpSmemT wsm[INTERACT_WARPS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int t = blockIdx.x * INTERACT_WARPS + wib;
  if (t >= P.ntasks) return;
  const int4 task = P.tasks[t];   // {leaf, first particle, count <= 32, -}
  bool v = lane < task.z;
  const int s = task.y + lane;
  const uint8_t st = (v && P.active) ? P.active[s] : (uint8_t)HS_ACTIVE;
  bool vc = v && st == HS_COARSE;
  if (v && P.active) v = st == HS_ACTIVE || st == HS_COARSE;
  if (!__any_sync(FULL_MASK, v)) return;
  DensOp op;
  op.xh = xh;
  op.vm = vm;
  op.nonly = out.nonly != 0;
  op.init(s, v);
  op.valid = v && !vc;
  traverse(op, P, task.x, smem[wib], smj[wib], smc[wib], wsm[wib], lane);
  if (__any_sync(FULL_MASK, vc)) {
    op.valid = op.act = vc;
    coarse_gather(op, P, task.x, smem[wib], smj[wib], smc[wib], wsm[wib], lane);
  }
  op.valid = v;
  if (v) {
    out.sf[s] = op.sf;
    out.acc0[s] = make_float4(op.smf, op.smqfp, op.sqfp, op.divs);
    out.s2[s] = op.sq2fpp;
    out.acc1[s] = make_float4(op.crx, op.cry, op.crz, __int_as_float(op.cnt));
  }
  long long nc = op.ncand;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nc += __shfl_xor_sync(FULL_MASK, nc, o);
  if (lane == 0 && P.ctr) {
    atomicAdd(&P.ctr[C_CAND], (unsigned long long)nc);
    atomicAdd(&P.ctr[C_TMP1], (unsigned long long)op.nseg);
    atomicAdd(&P.ctr[C_TMP2], (unsigned long long)op.nchunk);
    atomicMax(&P.ctr[C_MAXCH], (unsigned long long)op.nchunk);
    if (op.nchunk > 2000) atomicAdd(&P.ctr[C_HEAVY], (unsigned long long)op.nchunk);
    atomicMax(&P.ctr[C_MAXCH], (unsigned long long)op.nchunk);
    if (op.nchunk > 2000) atomicAdd(&P.ctr[C_HEAVY], (unsigned long long)op.nchunk);
  }
}

struct ForceOut {
  float* a;        // [n][3] caller order
  float* dudt;     // [n]
  float* vsig;     // [n] or null
  int* nnbr;       // [n] or null
  const uint32_t* perm;
  int64_t n_own;
};

__global__ void __launch_bounds__(INTERACT_WARPS * 32, SPH_FORCE_MINB) k_force(TravParams P, const float4* __restrict__ fx,
                                                               const float4* __restrict__ vm,
                                                               const float4* __restrict__ fs, float alpha,
                                                               const uint8_t* __restrict__ tau, ForceOut out) {
  __shared__ ForceOp::Src smem[INTERACT_WARPS][32];
  __shared__ int smj[INTERACT_WARPS][32];
  __shared__ int smc[INTERACT_WARPS][32];
  __shared__ WarpSmemT wsm[INTERACT_WARPS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int t = blockIdx.x * INTERACT_WARPS + wib;
  if (t >= P.ntasks) return;
  const int4 task = P.tasks[t];
  const int s = task.y + lane;
  const bool v = lane < task.z && out.perm[s] < out.n_own;   // halo particles are sources only
  if (!__any_sync(FULL_MASK, v)) return;
  ForceOp op;
  op.fx = fx;
  op.vm = vm;
  op.fs = fs;
  op.alpha = alpha;
  op.init(s, v);
  traverse(op, P, task.x, smem[wib], smj[wib], smc[wib], wsm[wib], lane);
  if (v) {
    const uint32_t p = out.perm[s];
    out.a[3 * (int64_t)p] = op.ax;
    out.a[3 * (int64_t)p + 1] = op.ay;
    out.a[3 * (int64_t)p + 2] = op.az;
    out.dudt[p] = op.du;
    if (out.vsig) out.vsig[p] = op.vsig;
    if (out.nnbr) out.nnbr[p] = op.cnt;
  }
  long long nc = op.ncand;
  long long nf = v ? op.cnt : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nc += __shfl_xor_sync(FULL_MASK, nc, o);
    nf += __shfl_xor_sync(FULL_MASK, nf, o);
  }
  if (lane == 0 && P.ctr) {
    atomicAdd(&P.ctr[C_CAND], (unsigned long long)nc);
    atomicAdd(&P.ctr[C_TMP1], (unsigned long long)op.nseg);
    atomicAdd(&P.ctr[C_TMP2], (unsigned long long)op.nchunk);
    atomicAdd(&P.ctr[C_NFORCE], (unsigned long long)nf);
  }
}

// ------------------------------------------------------------------ h update ------
// Safeguarded Newton iteration for N_i(h) = (32/3) sum_j f(r_ij/h) = n_ngb (Eq. 3,
// P:183-185; R3, R4), the step taken in log space: h' = h (n_ngb/N)^(1/nu) with
// nu = d ln N / d ln h = h N'/N from the same pass's sums (exact for N ~ h^nu, quadratic
// near the root like plain Newton). Steps are clamped to [h/2, 2h] and replaced by a
// bisection when they leave the bracket [lo, hi] of evaluated points. Converged iff
// |N - n_ngb| <= tol. A particle whose next h exceeds the h it was binned for (h_build)
// parks (state 2) until every other particle has converged; the cells are then rebuilt
// once for all parked particles.
__global__ void k_h_update(int64_t n, float4* __restrict__ xh, const float* __restrict__ hb,
                           float* __restrict__ lo, float* __restrict__ hi, uint8_t* __restrict__ state,
                           const double* __restrict__ sf, const float4* __restrict__ acc0,
                           const float* __restrict__ s2, float n_t, float tol, float coarse_cap, int nonly,
                           unsigned long long* ctr) {
  int unconv = 0, parked = 0, coarse = 0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    if (state[s] != HS_ACTIVE && state[s] != HS_COARSE) continue;
    const float h = xh[s].w;
    const double Nd = (32.0 / 3.0) * sf[s];
    const float N = (float)Nd;
    const float res = (float)(Nd - (double)n_t);
    if (fabsf(res) <= tol) {
      if (!nonly) state[s] = HS_DONE;            // N-only pass: keep h, evaluate the sums next pass
      else ++unconv;
      continue;
    }
    float l = lo[s], u = hi[s];
    if (res < 0.f) l = h;
    else u = h;
    lo[s] = l;
    hi[s] = u;
    if (u - l <= 4.f * (h * 1.1920929e-7f)) {   // bracket at fp32 resolution: stop
      if (!nonly) state[s] = HS_DONE;
      else ++unconv;
      continue;
    }
    // g(x) = ln N(e^x) - ln n_ngb with x = ln h:  g' = h N'/N,  g'' = g' + h^2 N''/N - g'^2,
    // h N' = -(32/3) S1, h^2 N'' = (32/3)(2 S1 + S2), S1 = sum q f'(q), S2 = sum q^2 f''(q)
    const float S1 = acc0[s].z, S2 = s2[s];
    const float g = __logf(N / n_t);
    const float g1 = -(32.f / 3.f) * S1 / N;
    const float g2 = g1 + (32.f / 3.f) * (2.f * S1 + S2) / N - g1 * g1;
    float dx;
    if (g1 > 0.25f) {
      dx = -g / g1;                                      // log-space Newton
      const float den = 2.f * g1 * g1 - g * g2;           // Halley (cubic convergence)
      if (den > 0.5f * g1 * g1) {
        const float dh = -2.f * g * g1 / den;
        if (fabsf(dh) <= 2.f * fabsf(dx)) dx = dh;
      }
    } else {
      dx = (res < 0.f) ? 0.6931472f : -0.6931472f;       // no neighbour yet: double / halve
    }
    float hn = h * __expf(dx);
    hn = fminf(fmaxf(hn, 0.5f * h), 2.f * h);
    if (!(hn > l && hn < u)) hn = 0.5f * (l + u);
    xh[s].w = hn;
    if (hn <= hb[s]) {
      state[s] = HS_ACTIVE;
      ++unconv;
    } else if (hn <= coarse_cap) {
      state[s] = HS_COARSE;
      ++unconv;
      ++coarse;
    } else {
      state[s] = HS_PARKED;
      ++parked;
    }
  }
  unconv = warp_sum_i(unconv);
  parked = warp_sum_i(parked);
  coarse = warp_sum_i(coarse);
  if ((threadIdx.x & 31) == 0) {
    if (unconv) atomicAdd(&ctr[C_UNCONV], (unsigned long long)unconv);
    if (parked) atomicAdd(&ctr[C_REBUILD], (unsigned long long)parked);
    if (coarse) atomicAdd(&ctr[C_TMP0], (unsigned long long)coarse);
  }
}

// particles whose final h exceeds the h their cells were built for
__global__ void k_count_loose(int64_t n, const float4* __restrict__ xh, const float* __restrict__ hb,
                              unsigned long long* ctr) {
  int cnt = 0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    cnt += xh[s].w > hb[s] ? 1 : 0;
  cnt = warp_sum_i(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&ctr[C_TMP0], (unsigned long long)cnt);
}

// tasks with at least one active lane (compaction flags)
__global__ void k_task_active(const int4* __restrict__ tasks, int ntasks,
                              const uint8_t* __restrict__ active, int* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (t >= ntasks) return;
  const int4 task = tasks[t];
  bool a = lane < task.z && active[task.y + lane] == HS_ACTIVE;
  bool any = __any_sync(FULL_MASK, a);
  if (lane == 0) flag[t] = any ? 1 : 0;
}

__global__ void k_task_compact(const int4* __restrict__ tasks, int ntasks, const int* __restrict__ flag,
                               const int* __restrict__ idx, int4* __restrict__ out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntasks && flag[t]) out[idx[t]] = tasks[t];
}

// ------------------------------------------------------------------ ghost --------
// P:770-781 "ghost": per-particle quantities between the density and force loops.
//   rho = (8/pi) h^-3 sum m f                      (Eq. 2)
//   Omega = -(sum m q f') / (3 sum m f)            (= 1 + h/(3 rho) drho/dh, identity)
//   P = (gamma-1) rho u,  c = sqrt(gamma (gamma-1) u),  A = P/(Omega rho^2)
//   div = sum m (f'/r) dv.dx / (h sum m f),  curl = -sum m (f'/r) dv x dx / (h sum m f)
//   f = |curl| / (|div| + |curl| + eps c/h)       (R10)
struct GhostOut {
  float* h;
  float* rho;
  float* omega;
  int* nnbr;
  float* div;
  float* curl;
  const uint32_t* perm;
  int64_t n_own;       // caller indices >= n_own are halo (source-only) particles
  float* h_o;          // caller-order state kept for the force loop: h
  float4* g_o;         //   {A, rho, c, f}
};

__global__ void k_ghost(int64_t n, const float4* __restrict__ xh, const float* __restrict__ u,
                        const double* __restrict__ sf, const float4* __restrict__ acc0,
                        const float4* __restrict__ acc1, float gamma, float beps, GhostOut out,
                        unsigned long long* ctr) {
  long long nd = 0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = out.perm[s];
    if (o >= out.n_own) continue;            // halo particle: its owner computes it
    const float4 p = xh[s];
    const float h = p.w, hinv = 1.0f / h;
    const float4 a0 = acc0[s], a1 = acc1[s];
    const float smf = a0.x;
    const float rho = SPH_CNORM * hinv * hinv * hinv * smf;
    const float omega = -a0.y / (3.f * smf);
    const float uu = u[s];
    const float P = (gamma - 1.f) * rho * uu;
    const float c = sqrtf(gamma * (gamma - 1.f) * uu);
    const float A = P / (omega * rho * rho);
    const float nrm = 1.0f / (h * smf);
    const float div = a0.w * nrm;
    const float cx = -a1.x * nrm, cy = -a1.y * nrm, cz = -a1.z * nrm;
    const float cn = sqrtf(cx * cx + cy * cy + cz * cz);
    const float fb = cn / (fabsf(div) + cn + beps * c * hinv);
    out.h_o[o] = h;
    out.g_o[o] = make_float4(A, rho, c, fb);
    const int cnt = __float_as_int(a1.w);
    nd += cnt;
    out.h[o] = h;
    out.rho[o] = rho;
    if (out.omega) out.omega[o] = omega;
    if (out.nnbr) out.nnbr[o] = cnt;
    if (out.div) out.div[o] = div;
    if (out.curl) {
      out.curl[3 * (int64_t)o] = cx;
      out.curl[3 * (int64_t)o + 1] = cy;
      out.curl[3 * (int64_t)o + 2] = cz;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nd += __shfl_xor_sync(FULL_MASK, nd, o);
  if ((threadIdx.x & 31) == 0 && nd) atomicAdd(&ctr[C_NDIR], (unsigned long long)nd);
}

// force inputs in the (possibly rebuilt) cell order from the caller-order state:
//   fx = {x, y, z, 1/h},  fs = {A (8/pi) h^-4, rho, c, f},  vm = {v, m}
__global__ void k_gather_force(const uint32_t* __restrict__ perm, int64_t n, const float4* __restrict__ xh,
                               const float* __restrict__ h_o, const float4* __restrict__ g_o,
                               const float* __restrict__ v, const float* __restrict__ m, float4* __restrict__ fx,
                               float4* __restrict__ fs, float4* __restrict__ vm) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[s];
    const float4 p = xh[s];
    const float hinv = 1.0f / h_o[o];
    const float h2i = hinv * hinv;
    const float4 g = g_o[o];
    fx[s] = make_float4(p.x, p.y, p.z, hinv);
    fs[s] = make_float4(g.x * SPH_CNORM * h2i * h2i, g.y, g.z, g.w);
    vm[s] = make_float4(v[3 * (int64_t)o], v[3 * (int64_t)o + 1], v[3 * (int64_t)o + 2], m[o]);
  }
}

// initial h-iteration state: owned particles active, halo (source-only) particles done
__global__ void k_init_state(const uint32_t* __restrict__ perm, int64_t n, int64_t n_own, uint8_t* __restrict__ st) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    st[s] = perm[s] < n_own ? HS_ACTIVE : HS_DONE;
}

// ------------------------------------------------------------------ slabs --------
// owned particles within `width` of the lower / upper face of the slab
// [lo, hi) (in x) are sent to the lower / upper neighbour rank as its halo (proxy cells of
// P:1065-1105). Flags here; compaction by scan keeps caller order.
__global__ void k_halo_flags(const float* __restrict__ x, int64_t n, float lo, float hi, float width,
                             int* __restrict__ flo, int* __restrict__ fhi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float xi = x[3 * i];
    flo[i] = (xi - lo < width) ? 1 : 0;
    fhi[i] = (hi - xi < width) ? 1 : 0;
  }
}

__global__ void k_compact_idx(const int* __restrict__ flag, const int* __restrict__ scan, int64_t n,
                              int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[scan[i]] = (int32_t)i;
}

__global__ void k_export_state(const int32_t* __restrict__ idx, int64_t k, const float* __restrict__ h_o,
                               const float4* __restrict__ g_o, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = idx[i];
    const float4 g = g_o[o];
    out[5 * i] = h_o[o];
    out[5 * i + 1] = g.x;
    out[5 * i + 2] = g.y;
    out[5 * i + 3] = g.z;
    out[5 * i + 4] = g.w;
  }
}

__global__ void k_import_state(const float* __restrict__ in, int64_t k, int64_t n_own, float* __restrict__ h_o,
                               float4* __restrict__ g_o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    h_o[n_own + i] = in[5 * i];
    g_o[n_own + i] = make_float4(in[5 * i + 1], in[5 * i + 2], in[5 * i + 3], in[5 * i + 4]);
  }
}

__global__ void k_x_hist(const float* __restrict__ x, int64_t n, float lo, float hi, int nb,
                         unsigned long long* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)floorf((x[3 * i] - lo) / (hi - lo) * nb);
    b = min(max(b, 0), nb - 1);
    atomicAdd(&hist[b], 1ull);
  }
}

// h_build for the force structure: the final h (plus rounding slack)
__global__ void k_force_hb(const float* __restrict__ h_o, int64_t n, float* __restrict__ hcur, float* __restrict__ hb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    hcur[i] = h_o[i];
    hb[i] = h_o[i] * (1.0f + 1e-5f);
  }
}

// ------------------------------------------------------------------ misc ---------
__global__ void k_validate_vmu(const float* __restrict__ v, const float* __restrict__ m, const float* __restrict__ u,
                               int64_t n, unsigned long long* ctr) {
  int err = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!isfinite(v[3 * i]) || !isfinite(v[3 * i + 1]) || !isfinite(v[3 * i + 2])) err |= ERRBIT_NONFINITE;
    if (!(m[i] > 0.f) || !isfinite(m[i])) err |= ERRBIT_MASS;
    if (!(u[i] > 0.f) || !isfinite(u[i])) err |= ERRBIT_U;
  }
  err = __reduce_or_sync(FULL_MASK, err);
  if ((threadIdx.x & 31) == 0 && err) atomicOr(&ctr[C_ERR], (unsigned long long)err);
}

__global__ void k_gather_vmu(const uint32_t* __restrict__ perm, int64_t n, const float* __restrict__ v,
                             const float* __restrict__ m, const float* __restrict__ u, float4* __restrict__ vm,
                             float* __restrict__ uc) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[s];
    vm[s] = make_float4(v[3 * (int64_t)p], v[3 * (int64_t)p + 1], v[3 * (int64_t)p + 2], m[p]);
    uc[s] = u[p];
  }
}

// scatter the iteration state back to caller order before a rebuild; h_build = h * margin
__global__ void k_scatter_state(const uint32_t* __restrict__ perm, int64_t n, const float4* __restrict__ xh,
                                const float* __restrict__ lo, const float* __restrict__ hi,
                                const uint8_t* __restrict__ state, float margin, float margin_parked, float hb_cap,
                                float* __restrict__ hcur_o, float* __restrict__ lo_o, float* __restrict__ hi_o,
                                float* __restrict__ hb_o) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[s];
    const float h = xh[s].w;
    hcur_o[p] = h;
    lo_o[p] = lo[s];
    hi_o[p] = hi[s];
    hb_o[p] = fminf(h * (state[s] == HS_PARKED ? margin_parked : margin), fmaxf(h, hb_cap));
  }
}

// carry the density sums and states of converged particles across a rebuild (the sums at a
// converged h do not depend on the cell structure); parked particles become active again
__global__ void k_scatter_sums(const uint32_t* __restrict__ perm, int64_t n, const uint8_t* __restrict__ state,
                               const double* __restrict__ sf, const float4* __restrict__ a0,
                               const float4* __restrict__ a1, uint8_t* __restrict__ state_o,
                               double* __restrict__ sf_o, float4* __restrict__ a0_o, float4* __restrict__ a1_o) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[s];
    const uint8_t st = state[s];
    state_o[p] = st == HS_DONE ? HS_DONE : HS_ACTIVE;   // coarse / parked particles resume normally
    if (st == HS_DONE) {
      sf_o[p] = sf[s];
      a0_o[p] = a0[s];
      a1_o[p] = a1[s];
    }
  }
}
__global__ void k_gather_sums(const uint32_t* __restrict__ perm, int64_t n, const uint8_t* __restrict__ state_o,
                              const double* __restrict__ sf_o, const float4* __restrict__ a0_o,
                              const float4* __restrict__ a1_o, uint8_t* __restrict__ state, double* __restrict__ sf,
                              float4* __restrict__ a0, float4* __restrict__ a1) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[s];
    const uint8_t st = state_o[p];
    state[s] = st;
    if (st == HS_DONE) {
      sf[s] = sf_o[p];
      a0[s] = a0_o[p];
      a1[s] = a1_o[p];
    }
  }
}

__global__ void k_fill_u8(uint8_t* p, int64_t n, uint8_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_fill_f(float* p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
// h state init from h0 (caller order): h_cur = h0, h_build = h0 * margin, bracket (0, inf)
__global__ void k_init_h(const float* __restrict__ h0, int64_t n, float margin, float hb_cap, float* __restrict__ hcur,
                         float* __restrict__ hb, float* __restrict__ lo, float* __restrict__ hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float h = h0[i];
    hcur[i] = h;
    hb[i] = fminf(h * margin, fmaxf(h, hb_cap));
    lo[i] = 0.f;
    hi[i] = INFINITY;
  }
}
__global__ void k_count_zero(const float* __restrict__ h, int64_t n, unsigned long long* ctr) {
  int z = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z += (h[i] == 0.f) ? 1 : 0;
  z = warp_sum_i(z);
  if ((threadIdx.x & 31) == 0 && z) atomicAdd(&ctr[C_TMP0], (unsigned long long)z);
}
// keep h0 where given, take the occupancy guess where h0 == 0
__global__ void k_merge_guess(const float* __restrict__ h0, int64_t n, float* __restrict__ guess) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (h0[i] > 0.f) guess[i] = h0[i];
}
