// hiter.cuh — the kernel function and the Newton/Halley step of the h iteration (Eq. 3,
// P:176-185), shared by the fused walk + solve (lists.cuh) and the stand-alone solve
// kernels (interact.cuh).
#pragma once
#include "common.cuh"

// per-particle states of the h iteration
#define HS_DONE 0
#define HS_ACTIVE 1
#define HS_REGROW 2   // needs a neighbour list for a new h_build (grown, or shrunk after overflow)

#define HS_OVF 3   // repeat overflow: needs an exactly sized list in the overflow pool
#ifndef HSOLVE_LONG
#define HSOLVE_LONG 256  // lists longer than this are solved by the whole warp
#endif

// counters of a solve (device, read once per round): unconverged, re-walks, pool, max iterations
#define HC_UNCONV 0
#define HC_REGROW 1
#define HC_OVF 2
#define HC_ITMAX 3
#define HC_EVALS 4   // entries summed by the h iteration (all evaluations, all rounds)
#define HC_N 5

// ------------------------------------------------------------------ kernel ------
// f(q) of the cubic spline (W = (8/pi) h^-3 f), its first and second derivative
__device__ __forceinline__ void spline(float q, float& f, float& fp, float& fpp) {
  const float t = 1.f - q;
  const bool in = q <= 0.5f;
  f = in ? fmaf(q * q, fmaf(6.f, q, -6.f), 1.f) : 2.f * t * t * t;
  fp = in ? q * fmaf(18.f, q, -12.f) : -6.f * t * t;
  fpp = in ? fmaf(36.f, q, -12.f) : 12.f * t;
}
__device__ __forceinline__ float spline_fp(float q) {
  const float t = 1.f - q;
  const float a = q * fmaf(18.f, q, -12.f), b = -6.f * t * t;
  return q <= 0.5f ? a : b;
}

// The neighbour lists hold r^2 (NB_STORE_R = 0: the square root is taken per entry and
// evaluation of the h sums, ~1.8 per entry) or r (NB_STORE_R = 1: taken when the walk tests
// the source, i.e. for every staged candidate on every lane, ~15x as many). Both give the
// same fp32 r = r^2 * rsqrt(r^2), so the two layouts agree bit for bit (C4: r^2 is 0.06 ms
// faster with the round-2 walk, profiles/round2/walk_experiments.md).
#ifndef NB_STORE_R
#define NB_STORE_R 0
#endif
__device__ __forceinline__ float nb_dist_of_r2(float r2) { return r2 * rsqrtf(fmaxf(r2, 1e-37f)); }
__device__ __forceinline__ float nb_stored(float r2) { return NB_STORE_R ? nb_dist_of_r2(r2) : r2; }
__device__ __forceinline__ float nb_r(float e) { return NB_STORE_R ? e : nb_dist_of_r2(e); }

// one iteration's sums over a list: S0 = sum f (fp64), S1 = sum q f', S2 = sum q^2 f''.
// Branch-free so the loads overlap: q is clamped to 1, where f = f' = f'' = 0 exactly.
#ifndef SPH_HSTEP_ACCEPT
#define SPH_HSTEP_ACCEPT 3e-3f
#endif
#ifndef NSUMS_UNROLL
#define NSUMS_UNROLL 4
#endif
// The lists are read with plain (weak, coherent) loads, never ld.global.nc: the fused solve
// reads lists its own warp wrote earlier in the same kernel (ordered by __syncwarp).
__device__ __forceinline__ void nsums(const float* r2l, int64_t stride, int e0, int e1, int estep,
                                      float hinv, double& S0, float& S1, float& S2) {
  int e = e0;
  const int64_t d = (int64_t)estep * stride;   // running pointer (no 64-bit product per load)
  const float* rp = r2l + (int64_t)e0 * stride;
  for (; e + (NSUMS_UNROLL - 1) * estep < e1; e += NSUMS_UNROLL * estep, rp += NSUMS_UNROLL * d) {
    float r2[NSUMS_UNROLL];
#pragma unroll
    for (int k = 0; k < NSUMS_UNROLL; ++k) r2[k] = rp[k * d];
#pragma unroll
    for (int k = 0; k < NSUMS_UNROLL; ++k) {
      const float q = fminf(nb_r(r2[k]) * hinv, 1.f);
      float f, fp, fpp;
      spline(q, f, fp, fpp);
      S0 += (double)f;
      S1 = fmaf(q, fp, S1);
      S2 = fmaf(q * q, fpp, S2);
    }
  }
  for (; e < e1; e += estep, rp += d) {
    const float r2 = *rp;
    const float q = fminf(nb_r(r2) * hinv, 1.f);
    float f, fp, fpp;
    spline(q, f, fp, fpp);
    S0 += (double)f;
    S1 = fmaf(q, fp, S1);
    S2 = fmaf(q * q, fpp, S2);
  }
}

// nsums for a contiguous, 16-byte aligned list (the per-particle rows of the slab): float4
// reads, same summation order as nsums.
__device__ __forceinline__ void nsums_row(const float* r2l, int e1, float hinv, double& S0, float& S1, float& S2) {
  const float4* r4 = reinterpret_cast<const float4*>(r2l);
  int e = 0;
  for (; e + 3 < e1; e += 4) {
    const float4 v = r4[e >> 2];
    const float r2[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float q = fminf(nb_r(r2[k]) * hinv, 1.f);
      float f, fp, fpp;
      spline(q, f, fp, fpp);
      S0 += (double)f;
      S1 = fmaf(q, fp, S1);
      S2 = fmaf(q * q, fpp, S2);
    }
  }
  for (; e < e1; ++e) {
    const float r2 = r2l[e];
    const float q = fminf(nb_r(r2) * hinv, 1.f);
    float f, fp, fpp;
    spline(q, f, fp, fpp);
    S0 += (double)f;
    S1 = fmaf(q, fp, S1);
    S2 = fmaf(q * q, fpp, S2);
  }
}

// nsums for one particle split over a segment of HSOLVE_SEG lanes (sub-lane sl): float4
// chunks sl, sl + SEG, ... of a 16-byte aligned contiguous row (the f of a chunk summed in
// fp32, then into the fp64 total), else entries sl, sl + SEG, ...
#ifndef HSOLVE_SEG
#define HSOLVE_SEG 4
#endif
#ifndef HSEG_PIPE
#define HSEG_PIPE 1     // load the next float4 chunk before summing this one (C4 build -0.07 ms)
#endif
__device__ __forceinline__ void nsums_seg(const float* r2l, int64_t stride, int cnt, int sl, float hinv, double& S0,
                                          float& S1, float& S2) {
  if (stride == 1 && ((reinterpret_cast<uintptr_t>(r2l) & 15) == 0)) {
    const float4* r4 = reinterpret_cast<const float4*>(r2l);
    const int nq = cnt >> 2;
#if HSEG_PIPE == 2
    float4 nxt = sl < nq ? r4[sl] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 nx2 = sl + HSOLVE_SEG < nq ? r4[sl + HSOLVE_SEG] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = sl; q < nq; q += HSOLVE_SEG) {
      const float4 v = nxt;
      nxt = nx2;
      if (q + 2 * HSOLVE_SEG < nq) nx2 = r4[q + 2 * HSOLVE_SEG];
#elif HSEG_PIPE
    float4 nxt = sl < nq ? r4[sl] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = sl; q < nq; q += HSOLVE_SEG) {
      const float4 v = nxt;
      if (q + HSOLVE_SEG < nq) nxt = r4[q + HSOLVE_SEG];   // the next chunk's load in flight
#else
    for (int q = sl; q < nq; q += HSOLVE_SEG) {
      const float4 v = r4[q];
#endif
      const float r2[4] = {v.x, v.y, v.z, v.w};
      float fs = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float qq = fminf(nb_r(r2[k]) * hinv, 1.f);
        float f, fp, fpp;
        spline(qq, f, fp, fpp);
        fs += f;
        S1 = fmaf(qq, fp, S1);
        S2 = fmaf(qq * qq, fpp, S2);
      }
      S0 += (double)fs;
    }
    for (int e = 4 * nq + sl; e < cnt; e += HSOLVE_SEG) {   // the last cnt % 4 entries
      const float qq = fminf(nb_r(r2l[e]) * hinv, 1.f);
      float f, fp, fpp;
      spline(qq, f, fp, fpp);
      S0 += (double)f;
      S1 = fmaf(qq, fp, S1);
      S2 = fmaf(qq * qq, fpp, S2);
    }
  } else {
    nsums(r2l, stride, sl, cnt, HSOLVE_SEG, hinv, S0, S1, S2);
  }
}

// One Newton/Halley update from the sums at h. Returns the new state: HS_DONE (converged),
// HS_ACTIVE (h updated, iterate), HS_REGROW (the new h lies beyond h_build).
__device__ __forceinline__ uint8_t hstep(double S0, float S1, float S2, float& h, float& hbs, float& l, float& u,
                                         float n_t, float tol, float margin, float hcap) {
  const double Nd = (32.0 / 3.0) * S0;
  const float N = (float)Nd;
  const float res = (float)(Nd - (double)n_t);
  if (fabsf(res) <= tol) return HS_DONE;
  if (res < 0.f) l = h;
  else u = h;
  if (u - l <= 4.f * (h * 1.1920929e-7f)) return HS_DONE;   // bracket at fp32 resolution
  // g' = h N'/N = -(32/3) S1 / N;  g'' = g' + (32/3)(2 S1 + S2)/N - g'^2
  const float g = __logf(N / n_t);
  const float g1 = -(32.f / 3.f) * S1 / N;
  const float g2 = g1 + (32.f / 3.f) * (2.f * S1 + S2) / N - g1 * g1;
  float dx;
  bool halley = false;
  if (g1 > 0.25f) {
    dx = -g / g1;                                     // log-space Newton
    const float den = 2.f * g1 * g1 - g * g2;          // Halley (cubic convergence)
    if (den > 0.5f * g1 * g1) {
      const float dh = -2.f * g * g1 / den;
      if (fabsf(dh) <= 2.f * fabsf(dx)) {
        dx = dh;
        halley = true;
      }
    }
  } else {
    dx = (res < 0.f) ? 0.6931472f : -0.6931472f;      // (almost) no neighbour: double / halve
  }
  float hn = h * __expf(dx);
  hn = fminf(fmaxf(hn, 0.5f * h), 2.f * h);
  const bool inb = hn > l && hn < u;
  if (!inb) hn = 0.5f * (l + fminf(u, 2.f * h));
  // floor at 2^-19 of the cap (~1e-6 L, below the fp32 resolution of distances in the box):
  // with more than 4 coincident particles N(h) > n_t for every h > 0 (no root);
  // such a particle stops here and is reported unconverged instead of underflowing
  hn = fminf(fmaxf(hn, hcap * 1.9073486e-6f), hcap);
  h = hn;
  if (hn > hbs) {                                     // the root lies beyond the list
    hbs = fminf(fminf(hn * margin, fmaxf(u, hn)), hcap);
    return HS_REGROW;
  }
  // A Halley step of |dx| <= SPH_HSTEP_ACCEPT leaves a residual of order |g3 / g1| dx^3 / 6
  // in ln N (g3 the third derivative; ~1e-7 N here), far inside tol: accept it without
  // another pass over the list. The density kernel re-checks N(h) at the final h from its
  // loop's sums, so a wrong acceptance is reported as unconverged, never silently kept.
  if (halley && inb && hn < hcap && fabsf(dx) <= SPH_HSTEP_ACCEPT) return HS_DONE;
  return HS_ACTIVE;
}


// One solve of the h iteration for the lanes of a warp (warp-collective): each active lane
// iterates on its own list (r2l, stride, cnt); lists longer than HSOLVE_LONG are summed by
// the whole warp, one particle at a time. A list holding more than K sources that is not
// in the pool was not recorded: h_build shrinks to hold ~K/2 sources and the particle is
// re-walked. fresh: the list was just recorded for this h_build (count-based start).
struct HLane {
  float h, hbs, l, u;
  uint8_t st;
  int it;
  long long ev;   // entries summed over all evaluations of N(h) (work of the iteration, Eq. 3)
};

__device__ __forceinline__ void warp_hsolve(bool act, const float* r2l, int64_t stride, int cnt, int K, bool pooled,
                                            bool fresh, HLane& H, float n_t, float tol, float margin, float hcap,
                                            int max_iter) {
  const int lane = threadIdx.x & 31;
  H.it = 0;
  if (act) {
    H.st = HS_ACTIVE;
    if (cnt > K && !pooled) {
      H.hbs = H.hbs * cbrtf(0.5f * (float)K / (float)cnt);
      H.h = fminf(H.h, H.hbs / margin);
      H.st = HS_REGROW;
    } else if (fresh && cnt > 0) {
      // start from the count within h_build: N(h) ~ C (h / h_build)^3 (locally uniform)
      const float he = H.hbs * cbrtf(n_t / (float)cnt);
      if (he > H.l && he < H.u && he <= H.hbs) H.h = he;
    }
    // N(h) is exact on the list only for h <= h_build: never start beyond it (a list
    // recorded below the initial h, e.g. a cold margin < 1, would otherwise set a false
    // lower bracket from a truncated sum)
    H.h = fminf(H.h, H.hbs);
  }
  const bool shortl = act && H.st == HS_ACTIVE && cnt <= HSOLVE_LONG;
#if HSOLVE_SEG > 1
  // Segments of HSOLVE_SEG lanes evaluate the sums of one particle each (the lane's own
  // particle loop left ~11 of 32 lanes busy: rows of different lengths, particles converging
  // after different numbers of steps). Each round takes the first 32 / HSOLVE_SEG pending
  // particles in lane order, one evaluation each; a particle stays pending while it iterates.
  {
    constexpr int NS = 32 / HSOLVE_SEG;
    const int seg = lane / HSOLVE_SEG, sl = lane % HSOLVE_SEG;
    unsigned pend = __ballot_sync(FULL_MASK, shortl && max_iter > 0);
    while (pend) {
      unsigned mm = pend;
      for (int k = 0; k < seg && mm; ++k) mm &= mm - 1;   // drop the first seg pending lanes
      const int owner = mm ? __ffs(mm) - 1 : -1;
      const int src = owner < 0 ? 0 : owner;
      const float* rp = reinterpret_cast<const float*>(__shfl_sync(FULL_MASK, (unsigned long long)r2l, src));
      const int64_t rs = __shfl_sync(FULL_MASK, stride, src);
      const int c = __shfl_sync(FULL_MASK, cnt, src);
      float h = __shfl_sync(FULL_MASK, H.h, src), hb = __shfl_sync(FULL_MASK, H.hbs, src);
      float l = __shfl_sync(FULL_MASK, H.l, src), u = __shfl_sync(FULL_MASK, H.u, src);
      double S0 = 0.0;
      float S1 = 0.f, S2 = 0.f;
      if (owner >= 0) nsums_seg(rp, rs, c, sl, 1.0f / h, S0, S1, S2);
#pragma unroll
      for (int o = 1; o < HSOLVE_SEG; o <<= 1) {
        S0 += __shfl_xor_sync(FULL_MASK, S0, o);
        S1 += __shfl_xor_sync(FULL_MASK, S1, o);
        S2 += __shfl_xor_sync(FULL_MASK, S2, o);
      }
      int st = HS_ACTIVE;
      if (owner >= 0) st = hstep(S0, S1, S2, h, hb, l, u, n_t, tol, margin, hcap);
      // back to the owners: a pending lane's segment is the number of pending lanes below it
      const int myseg = __popc(pend & lanemask_lt());
      const bool mine = ((pend >> lane) & 1u) && myseg < NS;
      const int from = mine ? myseg * HSOLVE_SEG : 0;
      h = __shfl_sync(FULL_MASK, h, from);
      hb = __shfl_sync(FULL_MASK, hb, from);
      l = __shfl_sync(FULL_MASK, l, from);
      u = __shfl_sync(FULL_MASK, u, from);
      st = __shfl_sync(FULL_MASK, st, from);
      bool again = ((pend >> lane) & 1u) != 0;
      if (mine) {
        H.h = h;
        H.hbs = hb;
        H.l = l;
        H.u = u;
        H.st = (uint8_t)st;
        H.ev += cnt;
        H.it += st == HS_REGROW ? 2 : 1;
        again = H.st == HS_ACTIVE && H.it < max_iter;
      }
      pend = __ballot_sync(FULL_MASK, again);
    }
  }
#else
  // one lane per particle, on its own row
  if (shortl) {
    for (; H.it < max_iter && H.st == HS_ACTIVE; ++H.it) {
      double S0 = 0.0;
      float S1 = 0.f, S2 = 0.f;
      if (stride == 1 && ((reinterpret_cast<uintptr_t>(r2l) & 15) == 0))
        nsums_row(r2l, cnt, 1.0f / H.h, S0, S1, S2);
      else
        nsums(r2l, stride, 0, cnt, 1, 1.0f / H.h, S0, S1, S2);
      H.ev += cnt;
      H.st = hstep(S0, S1, S2, H.h, H.hbs, H.l, H.u, n_t, tol, margin, hcap);
      if (H.st == HS_REGROW) ++H.it;
    }
  }
#endif
  unsigned lm = __ballot_sync(FULL_MASK, act && H.st == HS_ACTIVE && cnt > HSOLVE_LONG);
  while (lm) {
    const int t = __ffs(lm) - 1;
    lm &= lm - 1;
    const int tc = __shfl_sync(FULL_MASK, cnt, t);
    const int64_t tstr = __shfl_sync(FULL_MASK, stride, t);
    const float* tl = (const float*)__shfl_sync(FULL_MASK, (unsigned long long)r2l, t);
    float th = __shfl_sync(FULL_MASK, H.h, t), thb = __shfl_sync(FULL_MASK, H.hbs, t);
    float tlo = __shfl_sync(FULL_MASK, H.l, t), tu = __shfl_sync(FULL_MASK, H.u, t);
    uint8_t tst = HS_ACTIVE;
    int tit = 0;
    long long tev = 0;
    for (; tit < max_iter && tst == HS_ACTIVE; ++tit) {
      double S0 = 0.0;
      float S1 = 0.f, S2 = 0.f;
      nsums(tl, tstr, lane, tc, 32, 1.0f / th, S0, S1, S2);
      tev += tc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        S0 += __shfl_xor_sync(FULL_MASK, S0, o);
        S1 += __shfl_xor_sync(FULL_MASK, S1, o);
        S2 += __shfl_xor_sync(FULL_MASK, S2, o);
      }
      tst = hstep(S0, S1, S2, th, thb, tlo, tu, n_t, tol, margin, hcap);
      if (tst == HS_REGROW) ++tit;
    }
    if (lane == t) {
      H.h = th;
      H.hbs = thb;
      H.l = tlo;
      H.u = tu;
      H.st = tst;
      H.it = tit;
      H.ev += tev;
    }
  }
}

// warp totals of a solve into the round's counters
__device__ __forceinline__ void hsolve_count(bool act, const HLane& H, unsigned long long* hc) {
  const unsigned regrow = __ballot_sync(FULL_MASK, act && H.st == HS_REGROW);
  const unsigned unconv = __ballot_sync(FULL_MASK, act && H.st == HS_ACTIVE);
  const unsigned ovf = __ballot_sync(FULL_MASK, act && H.st == HS_OVF);
  const unsigned itmax = __reduce_max_sync(FULL_MASK, act ? (unsigned)H.it : 0u);
  unsigned long long ev = act ? (unsigned long long)H.ev : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(FULL_MASK, ev, o);
  if ((threadIdx.x & 31) == 0) {
    if (ev) atomicAdd(&hc[HC_EVALS], ev);
    if (regrow) atomicAdd(&hc[HC_REGROW], (unsigned long long)__popc(regrow));
    if (unconv) atomicAdd(&hc[HC_UNCONV], (unsigned long long)__popc(unconv));
    if (ovf) atomicAdd(&hc[HC_OVF], (unsigned long long)__popc(ovf));
    if (itmax) atomicMax(&hc[HC_ITMAX], (unsigned long long)itmax);
  }
}
