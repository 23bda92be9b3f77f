// interact.cuh — the density and force loops over the interaction lists (lists.cuh),
// the h update of the density iteration and the ghost step between the two loops.
//
// Work unit: one warp per target group (<= 32 particles of one leaf, lane = target i).
// The warp streams its group's list in stages of 32*ST sources: each lane loads one list
// entry and the source's data (float4, coalesced index reads, L2-resident gathers),
// shifts it into the group's frame and stages it in shared memory; then every lane
// tests every staged source against its own target (r < h_i, or r < max(h_i, h_j) for
// the force) into a hit mask, and runs the interaction body only for its hits.
// Gather form: a pair {i,j} is computed once from i's side and once from j's side (the
// paper's pair task updates both; here each target owns its accumulators, so
// there are no atomics and the sums are deterministic).
//
// Coordinates: positions are taken relative to the group's first particle o (in the
// group's frame, periodic images applied exactly: x - L for a source near L, o - L for a
// group near L; R19, H2), so the differences are exact or rounded at the scale of r.
#pragma once
#include "lists.cuh"

struct GroupLists {
  const int4* groups;
  const int64_t* off;
  const int* len;
  const uint32_t* list;
  int ngroups;
};

// ------------------------------------------------------------------ density ------
#ifndef DENS_WARPS
#define DENS_WARPS 8
#endif
#ifndef DENS_ST
#define DENS_ST 1          // staged sources per round: 32 * DENS_ST (tuned, tools/sweep.sh)
#endif

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
  // the force loop's cell-order inputs of the targets written here (null: k_gather_force
  // writes them): fx = {x, y, z, 1/h}, fs = {A (8/pi) h^-4, rho, c, f}, hr = h
  const float4* xh;
  float4* fx;
  float4* fs;
  float* hr;
};

// the density loop's epilogue is the ghost (a9): it writes the
// caller-order outputs and the force state, not the sums
struct DensOut {
  const float* u;
  float gamma, beps, n_t, tol_check;
  GhostOut g;
};

// a9 for one target from its density sums (k_density's epilogue)
__device__ __forceinline__ void ghost_one(const GhostOut& out, uint32_t o, int64_t s, float h, float uu, float smf,
                                          float smqfp, float divs, float crx, float cry, float crz, int cnt,
                                          float gamma, float beps) {
  const float hinv = 1.0f / h;
  const float rho = SPH_CNORM * hinv * hinv * hinv * smf;
  const float omega = -smqfp / (3.f * smf);
  const float P = (gamma - 1.f) * rho * uu;
  const float c = sqrtf(gamma * (gamma - 1.f) * uu);
  // Omega = 0 only without a neighbour at r > 0 inside h (R17): every G_i is then 0 and the
  // oracle's convention A_i G_i = 0 is kept by A_i = 0
  const float A = omega > 0.f ? P / (omega * rho * rho) : 0.f;
  const float nrm = 1.0f / (h * smf);
  const float div = divs * nrm;
  const float cx = -crx * nrm, cy = -cry * nrm, cz = -crz * nrm;
  const float cn = sqrtf(cx * cx + cy * cy + cz * cz);
  const float fb = cn / (fabsf(div) + cn + beps * c * hinv);
  out.h_o[o] = h;
  out.g_o[o] = make_float4(A, rho, c, fb);
  if (out.fx) {   // the same arithmetic as k_gather_force
    const float4 p = out.xh[s];
    const float h2i = hinv * hinv;
    out.fx[s] = make_float4(p.x, p.y, p.z, hinv);
    out.fs[s] = make_float4(A * SPH_CNORM * h2i * h2i, rho, c, fb);
    out.hr[s] = h;
  }
  if (out.h) out.h[o] = h;
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

// DIAG: also count (O8) borderline directed pairs |r / h_i - 1| <= SPH_BAND and coincident
// directed pairs (r = 0, j != i) into ctr[C_BORDER_D], ctr[C_COINC] (SPH_F_DIAGNOSTICS).
template <bool NONLY, bool DIAG = false>
#ifndef DENS_MINB
#define DENS_MINB 4     // 4 resident blocks of 8 warps: <= 64 registers (free: 72, 1: 89; both slower)
#endif
__global__ void __launch_bounds__(DENS_WARPS * 32, DENS_MINB) k_density(GroupLists G, const float4* __restrict__ xh,
                                                             const float4* __restrict__ vm,
                                                             const uint32_t* __restrict__ perm,
                                                             const uint8_t* __restrict__ tgt, float3 Lbox,
                                                             DensOut out, unsigned long long* ctr) {
  __shared__ float4 sp[DENS_WARPS][32 * DENS_ST];   // x, y, z (group frame), m
  __shared__ float4 sv[DENS_WARPS][32 * DENS_ST];   // vx, vy, vz, j (int bits)
  __shared__ __align__(8) float sxyz[DENS_WARPS][3][32 * DENS_ST];   // x, y, z again (SoA, packed tests)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gid = blockIdx.x * DENS_WARPS + wib;
  if (gid >= G.ngroups) return;
  const int4 grp = G.groups[gid];
  const int s = grp.y + lane;
  const bool act = lane < grp.z && tgt[s];   // halo and inactive particles: sources only
  if (!__any_sync(FULL_MASK, act)) return;
  const float L[3] = {Lbox.x, Lbox.y, Lbox.z};
  const float4 o4 = xh[grp.y];
  const float3 o = make_float3(o4.x, o4.y, o4.z);
  const float3 oL = make_float3(o4.x - L[0], o4.y - L[1], o4.z - L[2]);
  float xi = 0.f, yi = 0.f, zi = 0.f, hi = 0.f, vxi = 0.f, vyi = 0.f, vzi = 0.f;
  if (act) {
    const float4 p = xh[s];
    xi = p.x - o.x;
    yi = p.y - o.y;
    zi = p.z - o.z;
    hi = p.w;
    if (!NONLY) {
      const float4 q = vm[s];
      vxi = q.x;
      vyi = q.y;
      vzi = q.z;
    }
  }
  const float hi2 = act ? hi * hi : -1.f;
  const float hinv = act ? 1.0f / hi : 0.f;
  double sf = 0.0;
  float smf = 0.f, smqfp = 0.f, divs = 0.f, crx = 0.f, cry = 0.f, crz = 0.f;
  int cnt = 0;
  long long ncand = 0, nbord = 0, ncoin = 0;
  const int64_t off = G.off[gid];
  const int len = G.len[gid];
  float4* __restrict__ SP = sp[wib];
  float4* __restrict__ SV = sv[wib];
  // stage s takes entries s, s + nst, s + 2 nst, ...: every stage samples the whole list, so
  // the lanes' hit counts per stage are balanced (consecutive entries come from one cell)
  const int nst = (len + 32 * DENS_ST - 1) / (32 * DENS_ST);
  for (int stg = 0; stg < nst; ++stg) {
#pragma unroll
    for (int k = 0; k < DENS_ST; ++k) {
      const int e = stg + (32 * k + lane) * nst;
      float4 a = make_float4(1e30f, 1e30f, 1e30f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < len) {
        const uint32_t ent = G.list[off + e];
        const uint32_t j = ent & SPH_IDX_MASK;
        const float3 r = rel_pos(xh[j], ent >> SPH_IDX_BITS, o, oL, L);
        if (!NONLY) {
          b = vm[j];
          a = make_float4(r.x, r.y, r.z, b.w);
          b.w = __int_as_float((int)j);
        } else {
          a = make_float4(r.x, r.y, r.z, 0.f);
        }
      }
      SP[32 * k + lane] = a;
      SV[32 * k + lane] = b;
      sxyz[wib][0][32 * k + lane] = a.x;
      sxyz[wib][1][32 * k + lane] = a.y;
      sxyz[wib][2][32 * k + lane] = a.z;
    }
    __syncwarp();
    unsigned hm[DENS_ST];
#pragma unroll
    for (int k = 0; k < DENS_ST; ++k) {
      unsigned m = 0u;
      const float2* X2 = reinterpret_cast<const float2*>(sxyz[wib][0] + 32 * k);
      const float2* Y2 = reinterpret_cast<const float2*>(sxyz[wib][1] + 32 * k);
      const float2* Z2 = reinterpret_cast<const float2*>(sxyz[wib][2] + 32 * k);
#pragma unroll 8
      for (int t = 0; t < 16; ++t) {
        const float2 r2 = r2_pair(xi, yi, zi, X2[t], Y2[t], Z2[t]);
        m |= ((unsigned)(r2.x < hi2) | ((unsigned)(r2.y < hi2) << 1)) << (2 * t);
      }
      hm[k] = m;
      cnt += __popc(m);   // the directed neighbours (the target's own entry taken off below)
    }
    if (DIAG && act) {
      // same r^2 as the hit loop; the band |r^2 - h^2| <= 2 SPH_BAND h^2 is |r/h - 1| <= SPH_BAND
      for (int t = 0; t < 32 * DENS_ST; ++t) {
        const float4 q = SP[t];
        const float dx = xi - q.x, dy = yi - q.y, dz = zi - q.z;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        nbord += fabsf(r2 - hi2) <= 2.f * SPH_BAND * hi2 ? 1 : 0;
        ncoin += (r2 == 0.f && __float_as_int(SV[t].w) != s) ? 1 : 0;
      }
    }
    // interaction body for this lane's hits (sum f per stage in fp32, then into the fp64 sum)
    float sfs = 0.f;
    while (true) {
      int t = -1;
#pragma unroll
      for (int k = 0; k < DENS_ST; ++k) {
        if (t < 0 && hm[k]) {
          t = 32 * k + __ffs(hm[k]) - 1;
          hm[k] &= hm[k] - 1;
        }
      }
      if (t < 0) break;
      const float4 q = SP[t];
      const float dx = xi - q.x, dy = yi - q.y, dz = zi - q.z;
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float rinv = rsqrtf(fmaxf(r2, 1e-37f));   // r = 0 (self, duplicates): f' = 0 zeroes every r^-1 term
      const float qq = r2 * rinv * hinv;
      float f, fp, fpp;
      spline(qq, f, fp, fpp);   // (f'' is for the h iteration's sums only: unused here)
      sfs += f;
      const float qfp = qq * fp;
      if (!NONLY) {
        const float4 b = SV[t];
        const float mj = q.w;
        smf = fmaf(mj, f, smf);
        smqfp = fmaf(mj, qfp, smqfp);
        const float gf = mj * fp * rinv;
        const float dvx = b.x - vxi, dvy = b.y - vyi, dvz = b.z - vzi;
        divs = fmaf(gf, fmaf(dvx, dx, fmaf(dvy, dy, dvz * dz)), divs);
        crx = fmaf(gf, dvy * dz - dvz * dy, crx);
        cry = fmaf(gf, dvz * dx - dvx * dz, cry);
        crz = fmaf(gf, dvx * dy - dvy * dx, crz);
      }
    }
    sf += (double)sfs;
    __syncwarp();
  }
  // every staged entry was tested once (the stages partition the list); the target's own
  // entry (r = 0, image code 0) is in its group's list exactly once
  ncand = act ? len : 0;
  if (act) cnt -= 1;
  long long nd = 0, nbad = 0;
  if (act) {
    // the ghost (a9) in the epilogue: the caller-order outputs and the force state
    ghost_one(out.g, perm[s], s, hi, out.u[s], smf, smqfp, divs, crx, cry, crz, cnt, out.gamma, out.beps);
    nd = cnt;
    // the h iteration's convergence, re-checked from this loop's sum at the final h (R4)
    nbad = fabs((32.0 / 3.0) * sf - (double)out.n_t) > (double)out.tol_check ? 1 : 0;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) {
    ncand += __shfl_xor_sync(FULL_MASK, ncand, o2);
    nd += __shfl_xor_sync(FULL_MASK, nd, o2);
    nbad += __shfl_xor_sync(FULL_MASK, nbad, o2);
  }
  if (lane == 0 && ctr) {
    atomicAdd(&ctr[C_CAND], (unsigned long long)ncand);
    if (nd) atomicAdd(&ctr[C_NDIR], (unsigned long long)nd);
    if (nbad) atomicAdd(&ctr[C_UNCONV], (unsigned long long)nbad);
  }
  if (DIAG) {
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
      nbord += __shfl_xor_sync(FULL_MASK, nbord, o2);
      ncoin += __shfl_xor_sync(FULL_MASK, ncoin, o2);
    }
    if (lane == 0 && ctr) {
      atomicAdd(&ctr[C_BORDER_D], (unsigned long long)nbord);
      atomicAdd(&ctr[C_COINC], (unsigned long long)ncoin);
    }
  }
}

// ------------------------------------------------------------------ force --------
#ifndef FORCE_WARPS
#define FORCE_WARPS 4
#endif
#ifndef FORCE_ST
#define FORCE_ST 1
#endif

struct ForceOut {
  float* a;        // [n][3] caller order
  float* dudt;     // [n]
  float* vsig;     // [n] or null
  int* nnbr;       // [n] or null
  const uint32_t* perm;
  int64_t n_own;
  const uint8_t* tgt;   // cell order: 1 = target (owned and active)
};

// Eq. 4-5 + Monaghan-Balsara viscosity, symmetric pair scalar
//   T = A_i G_i + A_j G_j + (1/4) Pi (f_i + f_j)(G_i + G_j),  G = W_r / r,
//   a_i -= m_j T dx,  du_i += m_j (v_ij . dx) (A_i G_i + (1/8) Pi (f_i + f_j)(G_i + G_j)).
// fx = {x, y, z, 1/h}; fs = {A (8/pi) h^-4, rho, c, f}; vm = {v, m}.
// DIAG: also count borderline directed pairs |r / max(h_i, h_j) - 1| <= SPH_BAND (ctr[C_BORDER_F]).
template <bool DIAG = false>
#ifndef FORCE_MINB
#define FORCE_MINB 8    // 8 blocks of 4 warps: <= 64 registers, 32 resident warps
#endif
__global__ void __launch_bounds__(FORCE_WARPS * 32, FORCE_MINB) k_force(GroupLists G, const float4* __restrict__ fx,
                                                            const float4* __restrict__ vm,
                                                            const float4* __restrict__ fs, float alpha, float3 Lbox,
                                                            ForceOut out, unsigned long long* ctr) {
  __shared__ float4 sa[FORCE_WARPS][32 * FORCE_ST];   // x, y, z (group frame), 1/h_j
  __shared__ float4 sb[FORCE_WARPS][32 * FORCE_ST];   // v_j, m_j
  __shared__ float4 sc[FORCE_WARPS][32 * FORCE_ST];   // A~_j, rho_j, c_j, f_j
  __shared__ int sj[FORCE_WARPS][32 * FORCE_ST];
  __shared__ int sself[FORCE_WARPS][32];   // per target lane: its own particle's staged slot, or -1
  __shared__ __align__(8) float sxyzw[FORCE_WARPS][4][32 * FORCE_ST];   // x, y, z, 1/h^2 (SoA, packed tests)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gid = blockIdx.x * FORCE_WARPS + wib;
  if (gid >= G.ngroups) return;
  const int4 grp = G.groups[gid];
  const int s = grp.y + lane;
  const bool act = lane < grp.z && out.tgt[s];   // halo and inactive particles: sources only
  if (!__any_sync(FULL_MASK, act)) return;
  const float L[3] = {Lbox.x, Lbox.y, Lbox.z};
  const float4 o4 = fx[grp.y];
  const float3 o = make_float3(o4.x, o4.y, o4.z);
  const float3 oL = make_float3(o4.x - L[0], o4.y - L[1], o4.z - L[2]);
  float xi = 0.f, yi = 0.f, zi = 0.f, hinv = 0.f, vxi = 0.f, vyi = 0.f, vzi = 0.f;
  float At = 0.f, rhoi = 0.f, ci = 0.f, fi = 0.f;
  if (act) {
    const float4 p = fx[s], q = vm[s], w = fs[s];
    xi = p.x - o.x;
    yi = p.y - o.y;
    zi = p.z - o.z;
    hinv = p.w;
    vxi = q.x;
    vyi = q.y;
    vzi = q.z;
    At = w.x;
    rhoi = w.y;
    ci = w.z;
    fi = w.w;
  }
  const float hi = act ? 1.0f / hinv : 0.f;
  const float hi2 = act ? hi * hi : -1.f;
  const float h2i = hinv * hinv;
  const float hhat = SPH_CNORM * h2i * h2i;
  float ax = 0.f, ay = 0.f, az = 0.f, du = 0.f, vsig = 0.f;
  int cnt = 0;
  long long ncand = 0, nbord = 0;
  const int64_t off = G.off[gid];
  const int len = G.len[gid];
  float4* __restrict__ SA = sa[wib];
  float4* __restrict__ SB = sb[wib];
  float4* __restrict__ SC = sc[wib];
  int* __restrict__ SJ = sj[wib];
  // stage s takes entries s, s + nst, s + 2 nst, ...: every stage samples the whole list, so
  // the lanes' hit counts per stage are balanced (consecutive entries come from one cell)
  const int nst = (len + 32 * FORCE_ST - 1) / (32 * FORCE_ST);
  for (int stg = 0; stg < nst; ++stg) {
    sself[wib][lane] = -1;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < FORCE_ST; ++k) {
      const int e = stg + (32 * k + lane) * nst;
      float4 a = make_float4(1e30f, 1e30f, 1e30f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f), c = b;
      int jj = -1;
      if (e < len) {
        const uint32_t ent = G.list[off + e];
        const uint32_t j = ent & SPH_IDX_MASK;
        // the target's own particle (in its group's list with image code 0): its slot, so
        // the hit mask drops it once instead of a check per hit
        const int tl = (int)j - grp.y;
        if ((ent >> SPH_IDX_BITS) == 0 && tl >= 0 && tl < grp.z) sself[wib][tl] = 32 * k + lane;
        const float4 p = fx[j];
        const float3 r = rel_pos(p, ent >> SPH_IDX_BITS, o, oL, L);
        a = make_float4(r.x, r.y, r.z, p.w);
        b = vm[j];
        c = fs[j];
        jj = (int)j;
      }
      SA[32 * k + lane] = a;
      sxyzw[wib][0][32 * k + lane] = a.x;
      sxyzw[wib][1][32 * k + lane] = a.y;
      sxyzw[wib][2][32 * k + lane] = a.z;
      sxyzw[wib][3][32 * k + lane] = a.w * a.w;   // 1/h_j^2: the same product the hit body forms
      SB[32 * k + lane] = b;
      SC[32 * k + lane] = c;
      SJ[32 * k + lane] = jj;
    }
    __syncwarp();
    unsigned hm[FORCE_ST];
#pragma unroll
    for (int k = 0; k < FORCE_ST; ++k) {
      unsigned m = 0u;
      const float2* X2 = reinterpret_cast<const float2*>(sxyzw[wib][0] + 32 * k);
      const float2* Y2 = reinterpret_cast<const float2*>(sxyzw[wib][1] + 32 * k);
      const float2* Z2 = reinterpret_cast<const float2*>(sxyzw[wib][2] + 32 * k);
      const float2* W2 = reinterpret_cast<const float2*>(sxyzw[wib][3] + 32 * k);
#pragma unroll 8
      for (int t = 0; t < 16; ++t) {
        const float2 r2 = r2_pair(xi, yi, zi, X2[t], Y2[t], Z2[t]);
        const float2 hw2 = W2[t];
        const bool a0 = r2.x < hi2 || r2.x * hw2.x < 1.0f;
        const bool a1 = r2.y < hi2 || r2.y * hw2.y < 1.0f;
        m |= ((unsigned)a0 | ((unsigned)a1 << 1)) << (2 * t);
      }
      hm[k] = act ? m : 0u;
    }
    {
      const int sl = sself[wib][lane];
#if FORCE_ST == 1
      if (sl >= 0) hm[0] &= ~(1u << sl);
      cnt += __popc(hm[0]);
#else
#pragma unroll
      for (int k = 0; k < FORCE_ST; ++k)
        if (sl >= 0 && (sl >> 5) == k) hm[k] &= ~(1u << (sl & 31));
#pragma unroll
      for (int k = 0; k < FORCE_ST; ++k) cnt += __popc(hm[k]);
#endif
    }
    if (DIAG && act) {
      for (int t = 0; t < 32 * FORCE_ST; ++t) {
        const float4 qa = SA[t];
        if (SJ[t] < 0 || SJ[t] == s) continue;
        const float dx = xi - qa.x, dy = yi - qa.y, dz = zi - qa.z;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const float hm = fmaxf(hi, 1.0f / qa.w), hm2 = hm * hm;
        nbord += fabsf(r2 - hm2) <= 2.f * SPH_BAND * hm2 ? 1 : 0;
      }
    }
    while (true) {
      int t = -1;
#pragma unroll
      for (int k = 0; k < FORCE_ST; ++k) {
        if (t < 0 && hm[k]) {
          t = 32 * k + __ffs(hm[k]) - 1;
          hm[k] &= hm[k] - 1;
        }
      }
      if (t < 0) break;
      const float4 qa = SA[t], qb = SB[t], qc = SC[t];
      const float dx = xi - qa.x, dy = yi - qa.y, dz = zi - qa.z;
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float hjinv = qa.w;
      const float hj2i = hjinv * hjinv;
      const bool in_i = r2 < hi2;
      const bool in_j = r2 * hj2i < 1.0f;
      const float rinv = rsqrtf(fmaxf(r2, 1e-37f));   // r = 0 (self, duplicates): f' = 0 zeroes every r^-1 term
      const float r = r2 * rinv;
      const float fpi = in_i ? spline_fp(r * hinv) : 0.f;
      const float fpj = in_j ? spline_fp(r * hjinv) : 0.f;
      const float hhatj = SPH_CNORM * hj2i * hj2i;
      const float Gi = hhat * fpi * rinv;
      const float Gj = hhatj * fpj * rinv;
      const float vx = vxi - qb.x, vy = vyi - qb.y, vz = vzi - qb.z;
      const float vdx = fmaf(vx, dx, fmaf(vy, dy, vz * dz));
      const float w = fminf(0.f, vdx * rinv);
      const float cs = ci + qc.z - 3.f * w;
      const float Pi = __fdividef(-alpha * cs * w, rhoi + qc.y);
      const float V = Pi * (fi + qc.w) * (Gi + Gj);
      const float AGi = At * fpi * rinv;
      const float AGj = qc.x * fpj * rinv;
      const float T = AGi + AGj + 0.25f * V;
      const float mj = qb.w;
      const float mT = mj * T;
      ax = fmaf(-mT, dx, ax);
      ay = fmaf(-mT, dy, ay);
      az = fmaf(-mT, dz, az);
      du = fmaf(mj * vdx, AGi + 0.125f * V, du);
      vsig = fmaxf(vsig, cs);
    }
    __syncwarp();
  }
  ncand = act ? len : 0;   // every entry staged and tested once
  if (act) {
    const uint32_t p = out.perm[s];
    out.a[3 * (int64_t)p] = ax;
    out.a[3 * (int64_t)p + 1] = ay;
    out.a[3 * (int64_t)p + 2] = az;
    out.dudt[p] = du;
    if (out.vsig) out.vsig[p] = vsig;
    if (out.nnbr) out.nnbr[p] = cnt;
  }
  long long nf = act ? cnt : 0;
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) {
    ncand += __shfl_xor_sync(FULL_MASK, ncand, o2);
    nf += __shfl_xor_sync(FULL_MASK, nf, o2);
  }
  if (lane == 0 && ctr) {
    atomicAdd(&ctr[C_CAND], (unsigned long long)ncand);
    atomicAdd(&ctr[C_NFORCE], (unsigned long long)nf);
  }
  if (DIAG) {
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) nbord += __shfl_xor_sync(FULL_MASK, nbord, o2);
    if (lane == 0 && ctr) atomicAdd(&ctr[C_BORDER_F], (unsigned long long)nbord);
  }
}

// ------------------------------------------------------------------ symmetric force --
// The paper's pair update ("a pair ... updates both particles"; north_star item 4):
// every unordered pair {i, j} is evaluated ONCE, by its owner, and both particles are updated.
// Owner of the pair: the target group with the smaller index (a pair inside one group: the
// lower cell-order index; a pair with a source that is not a target, e.g. halo or inactive:
// the target's group). Each pair lies in both groups' interaction lists (the union criterion
// r < max(h_i, h_j) is symmetric), so every pair is found by its owner.
//   i side (the owner's lane): registers, written once per target (ia, idu, ivs, icnt);
//   j side: shared-memory slots per staged source (red.shared across the lanes that hit it),
//   one global red.add per slot and stage into ja / jdu / jvs / jcnt (cell order).
// k_force_sym_finish adds the two sides in the caller's order. Global float reductions are
// order-dependent, so unlike the gather kernel k_force this one is not bitwise deterministic.
struct ForceSym {
  const int* pgroup;   // cell order -> target group
  float4* ia;          // i side: a (xyz), du/dt
  float* ivs;
  int* icnt;
  float4* ja;          // j side (reductions)
  unsigned* jvs;       // v_sig bits (positive floats: integer max)
  int* jcnt;
};

template <bool DIAG>
__global__ void __launch_bounds__(FORCE_WARPS * 32, FORCE_MINB)
    k_force_sym(GroupLists G, const float4* __restrict__ fx, const float4* __restrict__ vm,
                const float4* __restrict__ fs, float alpha, float3 Lbox, ForceOut out, ForceSym Y,
                unsigned long long* ctr) {
  __shared__ float4 sa[FORCE_WARPS][32];   // x, y, z (group frame), 1/h_j
  __shared__ float4 sb[FORCE_WARPS][32];   // v_j, m_j
  __shared__ float4 sc[FORCE_WARPS][32];   // A~_j, rho_j, c_j, f_j
  __shared__ int sj[FORCE_WARPS][32];      // source index (cell order), -1 none
  __shared__ int sown[FORCE_WARPS][32];    // 1: the pair with this source is owned by any target of the group
  __shared__ float4 jacc[FORCE_WARPS][32]; // j-side sums of this stage
  __shared__ unsigned jvsm[FORCE_WARPS][32];
  __shared__ int jcn[FORCE_WARPS][32];
  __shared__ __align__(8) float sxyzw[FORCE_WARPS][4][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gid = blockIdx.x * FORCE_WARPS + wib;
  if (gid >= G.ngroups) return;
  const int4 grp = G.groups[gid];
  const int s = grp.y + lane;
  const bool act = lane < grp.z && out.tgt[s];
  if (!__any_sync(FULL_MASK, act)) return;
  const float L[3] = {Lbox.x, Lbox.y, Lbox.z};
  const float4 o4 = fx[grp.y];
  const float3 o = make_float3(o4.x, o4.y, o4.z);
  const float3 oL = make_float3(o4.x - L[0], o4.y - L[1], o4.z - L[2]);
  float xi = 0.f, yi = 0.f, zi = 0.f, hinv = 0.f, vxi = 0.f, vyi = 0.f, vzi = 0.f, mi = 0.f;
  float At = 0.f, rhoi = 0.f, ci = 0.f, fi = 0.f;
  if (act) {
    const float4 p = fx[s], q = vm[s], w = fs[s];
    xi = p.x - o.x;
    yi = p.y - o.y;
    zi = p.z - o.z;
    hinv = p.w;
    vxi = q.x;
    vyi = q.y;
    vzi = q.z;
    mi = q.w;
    At = w.x;
    rhoi = w.y;
    ci = w.z;
    fi = w.w;
  }
  const float hi = act ? 1.0f / hinv : 0.f;
  const float hi2 = act ? hi * hi : -1.f;
  const float h2i = hinv * hinv;
  const float hhat = SPH_CNORM * h2i * h2i;
  float ax = 0.f, ay = 0.f, az = 0.f, du = 0.f, vsig = 0.f;
  int cnt = 0;
  long long ncand = 0, nbord = 0;
  const int64_t off = G.off[gid];
  const int len = G.len[gid];
  const int nst = (len + 31) / 32;
  for (int stg = 0; stg < nst; ++stg) {
    const int e = stg + lane * nst;
    float4 a = make_float4(1e30f, 1e30f, 1e30f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f), c = b;
    int jj = -1, own = 0;
    if (e < len) {
      const uint32_t ent = G.list[off + e];
      const uint32_t j = ent & SPH_IDX_MASK;
      const float4 p = fx[j];
      const float3 r = rel_pos(p, ent >> SPH_IDX_BITS, o, oL, L);
      a = make_float4(r.x, r.y, r.z, p.w);
      b = vm[j];
      c = fs[j];
      jj = (int)j;
      // 2: every pair with j owned here; 1: owned for the targets below j in this group; 0: by j's group
      const int pj = Y.pgroup[j];
      own = (!out.tgt[j] || pj > gid) ? 2 : (pj == gid ? 1 : 0);
    }
    sa[wib][lane] = a;
    sxyzw[wib][0][lane] = a.x;
    sxyzw[wib][1][lane] = a.y;
    sxyzw[wib][2][lane] = a.z;
    sxyzw[wib][3][lane] = a.w * a.w;   // 1/h_j^2, as in k_force
    sb[wib][lane] = b;
    sc[wib][lane] = c;
    sj[wib][lane] = jj;
    sown[wib][lane] = own;
    jacc[wib][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
    jvsm[wib][lane] = 0u;
    jcn[wib][lane] = 0;
    __syncwarp();
    ncand += act ? min(32, (len - stg + nst - 1) / nst) : 0;
    unsigned hm = 0u;
    {
      const float2* X2 = reinterpret_cast<const float2*>(sxyzw[wib][0]);
      const float2* Y2 = reinterpret_cast<const float2*>(sxyzw[wib][1]);
      const float2* Z2 = reinterpret_cast<const float2*>(sxyzw[wib][2]);
      const float2* W2 = reinterpret_cast<const float2*>(sxyzw[wib][3]);
#pragma unroll 8
      for (int t = 0; t < 16; ++t) {
        const float2 r2 = r2_pair(xi, yi, zi, X2[t], Y2[t], Z2[t]);
        const float2 hw2 = W2[t];
        const bool a0 = r2.x < hi2 || r2.x * hw2.x < 1.0f;
        const bool a1 = r2.y < hi2 || r2.y * hw2.y < 1.0f;
        hm |= ((unsigned)a0 | ((unsigned)a1 << 1)) << (2 * t);
      }
      hm = act ? hm : 0u;
    }
    if (DIAG && act) {
      for (int t = 0; t < 32; ++t) {
        const float4 qa = sa[wib][t];
        if (sj[wib][t] < 0 || sj[wib][t] == s) continue;
        const float dx = xi - qa.x, dy = yi - qa.y, dz = zi - qa.z;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const float hmx = fmaxf(hi, 1.0f / qa.w), hm2 = hmx * hmx;
        nbord += fabsf(r2 - hm2) <= 2.f * SPH_BAND * hm2 ? 1 : 0;
      }
    }
    while (hm) {
      const int t = __ffs(hm) - 1;
      hm &= hm - 1;
      const int jt = sj[wib][t];
      const int ow = sown[wib][t];
      if (jt == s || ow == 0 || (ow == 1 && jt < s)) continue;   // self, or owned elsewhere
      const float4 qa = sa[wib][t], qb = sb[wib][t], qc = sc[wib][t];
      const float dx = xi - qa.x, dy = yi - qa.y, dz = zi - qa.z;
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float hjinv = qa.w;
      const float hj2i = hjinv * hjinv;
      const bool in_i = r2 < hi2;
      const bool in_j = r2 * hj2i < 1.0f;
      const float rinv = r2 > 0.f ? rsqrtf(r2) : 0.f;
      const float r = r2 * rinv;
      const float fpi = in_i ? spline_fp(r * hinv) : 0.f;
      const float fpj = in_j ? spline_fp(r * hjinv) : 0.f;
      const float hhatj = SPH_CNORM * hj2i * hj2i;
      const float Gi = hhat * fpi * rinv;
      const float Gj = hhatj * fpj * rinv;
      const float vx = vxi - qb.x, vy = vyi - qb.y, vz = vzi - qb.z;
      const float vdx = fmaf(vx, dx, fmaf(vy, dy, vz * dz));
      const float w = fminf(0.f, vdx * rinv);
      const float cs = ci + qc.z - 3.f * w;
      const float Pi = __fdividef(-alpha * cs * w, rhoi + qc.y);
      const float V = Pi * (fi + qc.w) * (Gi + Gj);
      const float AGi = At * fpi * rinv;
      const float AGj = qc.x * fpj * rinv;
      const float T = AGi + AGj + 0.25f * V;
      const float mj = qb.w;
      const float mT = mj * T;
      ax = fmaf(-mT, dx, ax);
      ay = fmaf(-mT, dy, ay);
      az = fmaf(-mT, dz, az);
      du = fmaf(mj * vdx, AGi + 0.125f * V, du);
      vsig = fmaxf(vsig, cs);
      cnt += 1;
      // j side: a_j += m_i T dx, du_j += m_i (v_ij . dx)(A_j G_j + V/8)
      const float miT = mi * T;
      atomicAdd(&jacc[wib][t].x, miT * dx);
      atomicAdd(&jacc[wib][t].y, miT * dy);
      atomicAdd(&jacc[wib][t].z, miT * dz);
      atomicAdd(&jacc[wib][t].w, mi * vdx * (AGj + 0.125f * V));
      atomicMax(&jvsm[wib][t], __float_as_uint(cs));
      atomicAdd(&jcn[wib][t], 1);
    }
    __syncwarp();
    // one global reduction per source slot of the stage that received a contribution
    if (jcn[wib][lane] > 0) {
      const int j = sj[wib][lane];
      const float4 q = jacc[wib][lane];
      atomicAdd(&Y.ja[j].x, q.x);
      atomicAdd(&Y.ja[j].y, q.y);
      atomicAdd(&Y.ja[j].z, q.z);
      atomicAdd(&Y.ja[j].w, q.w);
      atomicMax(&Y.jvs[j], jvsm[wib][lane]);
      atomicAdd(&Y.jcnt[j], jcn[wib][lane]);
    }
    __syncwarp();
  }
  if (act) {
    Y.ia[s] = make_float4(ax, ay, az, du);
    Y.ivs[s] = vsig;
    Y.icnt[s] = cnt;
  }
  long long nf = act ? cnt : 0;
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) {
    ncand += __shfl_xor_sync(FULL_MASK, ncand, o2);
    nf += __shfl_xor_sync(FULL_MASK, nf, o2);
  }
  if (lane == 0 && ctr) {
    atomicAdd(&ctr[C_CAND], (unsigned long long)ncand);
    atomicAdd(&ctr[C_NFORCE], 2ull * (unsigned long long)nf);   // each evaluated pair counts for both
  }
  if (DIAG) {
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) nbord += __shfl_xor_sync(FULL_MASK, nbord, o2);
    if (lane == 0 && ctr) atomicAdd(&ctr[C_BORDER_F], (unsigned long long)nbord);
  }
}

// both sides of the symmetric force into the caller's order (targets only)
__global__ void k_force_sym_finish(const uint32_t* __restrict__ perm, int64_t n, const uint8_t* __restrict__ tgt,
                                   ForceSym Y, ForceOut out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    if (!tgt[s]) continue;
    const uint32_t p = perm[s];
    const float4 a = Y.ia[s], b = Y.ja[s];
    out.a[3 * (int64_t)p] = a.x + b.x;
    out.a[3 * (int64_t)p + 1] = a.y + b.y;
    out.a[3 * (int64_t)p + 2] = a.z + b.z;
    out.dudt[p] = a.w + b.w;
    if (out.vsig) out.vsig[p] = fmaxf(Y.ivs[s], __uint_as_float(Y.jvs[s]));
    if (out.nnbr) out.nnbr[p] = Y.icnt[s] + Y.jcnt[s];
  }
}

__global__ void k_pgroup(const int4* __restrict__ groups, int ng, int* __restrict__ pgroup) {
  const int lane = threadIdx.x & 31;
  const int g = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (g >= ng) return;
  const int4 gr = groups[g];
  if (lane < gr.z) pgroup[gr.y + lane] = g;
}

// ------------------------------------------------------------------ h solve -------
// The h iteration of Eq. 3 (R3, R4) for every particle on its own neighbour
// list: the squared distances r^2 < h_build^2 recorded by the NB walk (lists.cuh). For any
// h <= h_build, N(h) = (32/3) sum_{r < h} f(r/h) (self term included, R2) is exact on the
// list, so the whole iteration runs here without further sweeps of the cells:
//   x = ln h, g(x) = ln N - ln n_ngb, g' = h N'/N, g'' from the same sums;
//   Newton step in log space with Halley's correction, clamped to [h/2, 2h] and replaced
//   by a bisection when it leaves the bracket [lo, hi] of evaluated points;
//   converged iff |N - n_ngb| <= tol (or the bracket is at fp32 resolution).
// A step beyond h_build (the root lies outside the list) sets h_build = h * margin and
// state HS_REGROW: the walk re-records this particle's list before the next round. A list
// longer than K lives in the overflow pool (contiguous, exactly sized; lists.cuh).
#define HSOLVE_WARPS 8

__global__ void __launch_bounds__(HSOLVE_WARPS * 32) k_hsolve(const int4* __restrict__ groups, int ngroups,
                                                              float4* __restrict__ xh, float* __restrict__ hb,
                                                              float* __restrict__ lo_a, float* __restrict__ hi_a,
                                                              uint8_t* __restrict__ state,
                                                              const float* __restrict__ nb_r2,
                                                              const int* __restrict__ nb_cnt, int K,
                                                              const int64_t* __restrict__ ovf_off,
                                                              const float* __restrict__ ovf, float n_t,
                                                              float tol, float margin, float hcap, int max_iter,
                                                              unsigned long long* hc) {
  const int lane = threadIdx.x & 31;
  const int gid = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (gid >= ngroups) return;
  const int4 grp = groups[gid];
  const int s = grp.y + lane;
  // particles with a list in the overflow pool are solved by k_hsolve_pool
  const bool act = lane < grp.z && state[s] == HS_ACTIVE && ovf_off[s] < 0;
  if (!__any_sync(FULL_MASK, act)) return;
  HLane H;
  H.h = H.hbs = H.l = H.u = 0.f;
  H.ev = 0;
  H.st = HS_DONE;
  int cnt = 0;
  if (act) {
    cnt = nb_cnt[s];
    H.h = xh[s].w;
    H.hbs = hb[s];
    H.l = lo_a[s];
    H.u = hi_a[s];
  }
  warp_hsolve(act, nb_r2 + (NB_ROWS ? (int64_t)s * K : (int64_t)grp.y * K + lane), NB_ROWS ? 1 : grp.z, cnt, K, false,
              false, H, n_t, tol, margin, hcap,
              max_iter);
  if (act) {
    xh[s].w = H.h;
    hb[s] = H.hbs;
    lo_a[s] = H.l;
    hi_a[s] = H.u;
    state[s] = H.st;
  }
  hsolve_count(act, H, hc);
}

// The h iteration for particles whose list lives in the overflow pool (long, contiguous):
// one warp per particle, the sums reduced across the warp each iteration.
__global__ void __launch_bounds__(HSOLVE_WARPS * 32) k_hsolve_pool(const int* __restrict__ idx, int nidx,
                                                                   float4* __restrict__ xh, float* __restrict__ hb,
                                                                   float* __restrict__ lo_a, float* __restrict__ hi_a,
                                                                   uint8_t* __restrict__ state,
                                                                   const int* __restrict__ nb_cnt,
                                                                   const int64_t* __restrict__ ovf_off,
                                                                   const float* __restrict__ ovf, float n_t, float tol,
                                                                   float margin, float hcap, int max_iter,
                                                                   unsigned long long* hc) {
  const int lane = threadIdx.x & 31;
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (w >= nidx) return;
  const int s = idx[w];
  const int64_t oo = ovf_off[s];
  if (state[s] != HS_ACTIVE || oo < 0) return;
  const int cnt = nb_cnt[s];
  const float* r2l = ovf + oo;
  float h = xh[s].w, hbs = hb[s], l = lo_a[s], u = hi_a[s];
  uint8_t st = HS_ACTIVE;
  int it = 0;
  unsigned long long ev = 0;
  for (; it < max_iter && st == HS_ACTIVE; ++it) {
    double S0 = 0.0;
    float S1 = 0.f, S2 = 0.f;
    nsums(r2l, 1, lane, cnt, 32, 1.0f / h, S0, S1, S2);
    ev += cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      S0 += __shfl_xor_sync(FULL_MASK, S0, o);
      S1 += __shfl_xor_sync(FULL_MASK, S1, o);
      S2 += __shfl_xor_sync(FULL_MASK, S2, o);
    }
    st = hstep(S0, S1, S2, h, hbs, l, u, n_t, tol, margin, hcap);
    if (st == HS_REGROW) ++it;
  }
  if (lane == 0) {
    xh[s].w = h;
    hb[s] = hbs;
    lo_a[s] = l;
    hi_a[s] = u;
    state[s] = st;
    if (st == HS_REGROW) atomicAdd(&hc[HC_REGROW], 1ull);
    if (st == HS_ACTIVE) atomicAdd(&hc[HC_UNCONV], 1ull);
    atomicMax(&hc[HC_ITMAX], (unsigned long long)it);
    atomicAdd(&hc[HC_EVALS], ev);
  }
}

// UNION-walk reach in the density phase: the h of owned particles (halo h unknown: 0)
__global__ void k_reach_owned(const uint32_t* __restrict__ perm, int64_t n, int64_t n_own,
                              const float4* __restrict__ xh, float* __restrict__ hr) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    hr[s] = perm[s] < n_own ? xh[s].w : 0.f;
}

// HS_REGROW -> HS_ACTIVE once the new lists are recorded
__global__ void k_state_swap(uint8_t* __restrict__ st, int64_t n, uint8_t from, uint8_t to) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    if (st[s] == from) st[s] = to;
}

// ------------------------------------------------------------------ ghost --------
// P:770-781 "ghost": per-particle quantities between the density and force loops.
//   rho = (8/pi) h^-3 sum m f                      (Eq. 2)
//   Omega = -(sum m q f') / (3 sum m f)            (= 1 + h/(3 rho) drho/dh, identity)
//   P = (gamma-1) rho u,  c = sqrt(gamma (gamma-1) u),  A = P/(Omega rho^2)
//   div = sum m (f'/r) dv.dx / (h sum m f),  curl = -sum m (f'/r) dv x dx / (h sum m f)
//   f = |curl| / (|div| + |curl| + eps c/h)       (R10)

// force inputs in cell order from the caller-order state (owned: the ghost; halo: imported):
//   fx = {x, y, z, 1/h},  fs = {A (8/pi) h^-4, rho, c, f},  hr = h (the force list reach)
__global__ void k_gather_force(const uint32_t* __restrict__ perm, int64_t n, const float4* __restrict__ xh,
                               const float* __restrict__ h_o, const float4* __restrict__ g_o,
                               float4* __restrict__ fx, float4* __restrict__ fs, float* __restrict__ hr) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[s];
    const float4 p = xh[s];
    const float h = h_o[o];
    const float hinv = 1.0f / h;
    const float h2i = hinv * hinv;
    const float4 g = g_o[o];
    fx[s] = make_float4(p.x, p.y, p.z, hinv);
    fs[s] = make_float4(g.x * SPH_CNORM * h2i * h2i, g.y, g.z, g.w);
    hr[s] = h;
  }
}

// iteration state in cell order: owned particles active (bracket (0, inf), h_build =
// h * margin), halo (source-only) particles done
__global__ void k_init_iter(const uint8_t* __restrict__ tgt, int64_t n, const float4* __restrict__ xh,
                            float margin, float hcap, uint8_t* __restrict__ st, float* __restrict__ hb,
                            float* __restrict__ lo, float* __restrict__ hi) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const bool own = tgt[s] != 0;   // targets iterate; halo and inactive particles keep their h
    st[s] = own ? HS_ACTIVE : HS_DONE;
    if (hb) hb[s] = own ? fminf(xh[s].w * margin, hcap) : 0.f;
    lo[s] = 0.f;
    hi[s] = INFINITY;
  }
}

// ------------------------------------------------------------------ slabs --------
// owned particles within `width` of the lower / upper face of the slab
// [lo, hi) (in x) are sent to the lower / upper neighbour rank as its halo (proxy cells of
// P:1065-1105). Flags here; compaction by scan keeps caller order.
// width > 0: within width of the faces (halo); width == 0: outside [lo, hi) (slab leavers)
__global__ void k_halo_flags(const float* __restrict__ x, int64_t n, float lo, float hi, float width,
                             int* __restrict__ flo, int* __restrict__ fhi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float xi = x[3 * i];
    if (width > 0.f) {
      flo[i] = (xi - lo < width) ? 1 : 0;
      fhi[i] = (hi - xi < width) ? 1 : 0;
    } else {
      flo[i] = (xi < lo) ? 1 : 0;
      fhi[i] = (xi >= hi) ? 1 : 0;
    }
  }
}

// first-exchange rows {x, v, m, u, h0} of the listed owned particles (the
// particles a proxy cell needs)
__global__ void k_halo_pack(const float* __restrict__ x, const float* __restrict__ v, const float* __restrict__ m,
                            const float* __restrict__ u, const float* __restrict__ h0, const int32_t* __restrict__ idx,
                            int64_t k, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = idx[i];
    float* r = out + 9 * i;
    r[0] = x[3 * o];
    r[1] = x[3 * o + 1];
    r[2] = x[3 * o + 2];
    r[3] = v[3 * o];
    r[4] = v[3 * o + 1];
    r[5] = v[3 * o + 2];
    r[6] = m[o];
    r[7] = u[o];
    r[8] = h0 ? h0[o] : 0.f;
  }
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

// the halo width the owned particles need (a proxy cell holds every foreign
// particle an owned one interacts with): the largest h of an owned particle within h of a
// slab face. A foreign j must be in the halo iff some owned i has r_ij < max(h_i, h_j); both
// cases put the particle with the larger h within that h of the face, so the max over both
// ranks of this quantity bounds the distance beyond the face any partner lies at.
__global__ void k_hface(const uint32_t* __restrict__ perm, const float4* __restrict__ xh, int64_t n, int64_t n_own,
                        float lo, float hi, unsigned long long* ctr) {
  unsigned mx = 0u;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    if (perm[s] >= n_own) continue;
    const float4 p = xh[s];
    if (p.x - lo < p.w || hi - p.x < p.w) mx = max(mx, __float_as_uint(p.w));
  }
  mx = __reduce_max_sync(FULL_MASK, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&ctr[C_HMAXBITS], (unsigned long long)mx);
}

// work-weighted histogram (integer work units: exact, order-independent sums)
__global__ void k_x_hist_w(const float* __restrict__ x, const int32_t* __restrict__ w, int64_t n, float lo, float hi,
                           int nb, unsigned long long* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)floorf((x[3 * i] - lo) / (hi - lo) * nb);
    b = min(max(b, 0), nb - 1);
    atomicAdd(&hist[b], (unsigned long long)max(w[i], 0));
  }
}

// ------------------------------------------------------------------ misc ---------
// v, m, u checked (finite; m, u > 0) and packed in caller order as float4 {v, m} and u in
// one coalesced pass, so the permute below gathers one 16-byte record (+ u) per particle
__global__ void k_validate_pack_vmu(const float* __restrict__ v, const float* __restrict__ m,
                                    const float* __restrict__ u, int64_t n, float4* __restrict__ vmc,
                                    unsigned long long* ctr) {
  int err = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float a = v[3 * i], b = v[3 * i + 1], c = v[3 * i + 2], mm = m[i], uu = u[i];
    if (!isfinite(a) || !isfinite(b) || !isfinite(c)) err |= ERRBIT_NONFINITE;
    if (!(mm > 0.f) || !isfinite(mm)) err |= ERRBIT_MASS;
    if (!(uu > 0.f) || !isfinite(uu)) err |= ERRBIT_U;
    vmc[i] = make_float4(a, b, c, mm);
  }
  err = __reduce_or_sync(FULL_MASK, err);
  if ((threadIdx.x & 31) == 0 && err) atomicOr(&ctr[C_ERR], (unsigned long long)err);
}

__global__ void k_gather_vmu(const uint32_t* __restrict__ perm, int64_t n, const float4* __restrict__ vmc,
                             const float* __restrict__ u, float4* __restrict__ vm, float* __restrict__ uc) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[s];
    vm[s] = vmc[p];
    uc[s] = u[p];
  }
}

// h of the owned particles in caller order (the early copy-back of sph_density)
__global__ void k_scatter_h_own(const uint32_t* __restrict__ perm, int64_t n, int64_t n_own,
                                const float4* __restrict__ xh, float* __restrict__ h_o) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[s];
    if (o < n_own) h_o[o] = xh[s].w;
  }
}

// h in caller order from cell order (the initial-guess call)
__global__ void k_scatter_h(const uint32_t* __restrict__ perm, int64_t n, const float4* __restrict__ xh,
                            float* __restrict__ h_o) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    h_o[perm[s]] = xh[s].w;
}

// cell-order target flags: owned (caller index < n_own) and active (caller mask, or all)
__global__ void k_make_tgt(const uint32_t* __restrict__ perm, int64_t n, int64_t n_own,
                           const uint8_t* __restrict__ active, uint8_t* __restrict__ tgt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[s];
    tgt[s] = (o < n_own && (!active || active[o])) ? 1 : 0;
  }
}

// Neighbour minimum for the time-step limiter (individual time steps): for
// every target i of the last force loop and every j in its interaction list with
// r_ij < max(h_i, h_j) (the force pairs): out[j] = min(out[j], val[i]) in the
// caller's order (positive floats as bits: atomicMin is order-independent, so the result is
// deterministic). Warp per group, lane = target; sources staged 32 at a time.
__global__ void __launch_bounds__(256) k_scatter_min(GroupLists G, const float4* __restrict__ fx,
                                                     const uint32_t* __restrict__ perm,
                                                     const uint8_t* __restrict__ tgt, const float* __restrict__ val,
                                                     float3 Lbox, unsigned* __restrict__ out_bits) {
  __shared__ float4 sa[8][32];
  __shared__ unsigned so[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gid = blockIdx.x * 8 + wib;
  if (gid >= G.ngroups) return;
  const int4 grp = G.groups[gid];
  const int s = grp.y + lane;
  const bool act = lane < grp.z && tgt[s];
  if (!__any_sync(FULL_MASK, act)) return;
  const float L[3] = {Lbox.x, Lbox.y, Lbox.z};
  const float4 o4 = fx[grp.y];
  const float3 o = make_float3(o4.x, o4.y, o4.z);
  const float3 oL = make_float3(o4.x - L[0], o4.y - L[1], o4.z - L[2]);
  float xi = 0.f, yi = 0.f, zi = 0.f, hi2 = -1.f;
  unsigned vi = 0x7f800000u;
  if (act) {
    const float4 p = fx[s];
    xi = p.x - o.x;
    yi = p.y - o.y;
    zi = p.z - o.z;
    const float hi = 1.0f / p.w;
    hi2 = hi * hi;
    vi = __float_as_uint(val[perm[s]]);
  }
  const int64_t off = G.off[gid];
  const int len = G.len[gid];
  for (int b0 = 0; b0 < len; b0 += 32) {
    const int e = b0 + lane;
    float4 a = make_float4(1e30f, 1e30f, 1e30f, 0.f);
    unsigned oj = 0xffffffffu;
    if (e < len) {
      const uint32_t ent = G.list[off + e];
      const uint32_t j = ent & SPH_IDX_MASK;
      const float4 p = fx[j];
      const float3 r = rel_pos(p, ent >> SPH_IDX_BITS, o, oL, L);
      a = make_float4(r.x, r.y, r.z, p.w);
      oj = perm[j];
    }
    sa[wib][lane] = a;
    so[wib][lane] = oj;
    __syncwarp();
    // per source (lane = source): the smallest value of the targets that reach it
    unsigned best = 0x7f800000u;
    const float4 q = sa[wib][lane];
    for (int t = 0; t < 32; ++t) {
      const float tx = __shfl_sync(FULL_MASK, xi, t), ty = __shfl_sync(FULL_MASK, yi, t);
      const float tz = __shfl_sync(FULL_MASK, zi, t), th2 = __shfl_sync(FULL_MASK, hi2, t);
      const unsigned tv = __shfl_sync(FULL_MASK, vi, t);
      const float dx = tx - q.x, dy = ty - q.y, dz = tz - q.z;
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      if (th2 >= 0.f && (r2 < th2 || r2 * (q.w * q.w) < 1.0f)) best = min(best, tv);
    }
    const unsigned ob = so[wib][lane];
    if (ob != 0xffffffffu && best != 0x7f800000u) atomicMin(&out_bits[ob], best);
    __syncwarp();
  }
}
