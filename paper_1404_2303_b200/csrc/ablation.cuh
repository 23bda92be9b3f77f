// ablation.cuh — the paper's own cell-pair loops, for the sorted-vs-naive ablation
// (section 3.3). Not on the hot path.
//
// Cells: a uniform periodic grid of edge >= max h (one level), particles in cell
// order (counting sort). Pairs: each cell with itself and its 13 forward neighbours (
// the other 13 are the same pairs seen from the other side). Per cell pair, the density sums
// rho_i = sum_j m_j W(r_ij, h_i) of both cells (Eq. 2, each direction with its own h):
//   naive: every particle of A against every particle of B;
//   sorted (R6, R7): A and B presorted along the pair's axis d (13 canonical
//          directions; only forward offsets are enumerated, so the stored order is the one
//          needed, R20); sweep 1 takes each i of A against the j of B in ascending projection
//          until r_i + h_i < r_j; sweep 2 each j of B against the i of A in descending
//          projection until r_i < r_j - h_j, keeping only r >= h_i there (R6: the
//          complement of sweep 1, so a pair at r == h_i exactly is never lost).
// Each found pair updates both densities with their own h (the paper's "compute interaction").
// One warp per cell pair, lanes over the sweeping side's particles (chunks of 32). rho is
// reduced with float atomics (order-dependent; the ablation checks it against sph_density's
// rho at 1e-5). Counters: distance tests, tests per direction class (face / edge / corner), and
// the window passes (pairs whose projected separation is inside the window, the paper's
// 16.2 / 3.6 % for edge / corner neighbours of cells of edge h, R9).
#pragma once
#include "common.cuh"

// ablation counters (int64 slots)
#define AB_TESTS 0       // distance tests
#define AB_HITS 1        // directed contributions r < h_i (j != i)
#define AB_PAIRS_F 2     // particle pairs (nA x nB) of face / edge / corner cell pairs
#define AB_PAIRS_E 3
#define AB_PAIRS_C 4
#define AB_PASS_F 5      // sweep-1 window passes (p_j - p_i < h_i) of face / edge / corner cell pairs
#define AB_PASS_E 6
#define AB_PASS_C 7
#define AB_INR_F 8       // sweep-1 in-range (r < h_i) of face / edge / corner cell pairs
#define AB_INR_E 9
#define AB_INR_C 10
#define AB_N 11

__device__ __forceinline__ int dir_class(int k) {   // offset k: number of non-zero components
  return (off_x(k) != 0) + (off_y(k) != 0) + (off_z(k) != 0);
}

// cell of each particle (cell order of the build; positions xh) and per-cell counts
__global__ void k_ab_cells(const float4* __restrict__ xh, int64_t n, int nx, int ny, int nz, float ix, float iy,
                           float iz, int* __restrict__ cell, int* __restrict__ ccount) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const float4 p = xh[s];
    int cx = (int)floorf(p.x * ix), cy = (int)floorf(p.y * iy), cz = (int)floorf(p.z * iz);
    cx = ((cx % nx) + nx) % nx;
    cy = ((cy % ny) + ny) % ny;
    cz = ((cz % nz) + nz) % nz;
    const int c = cx + nx * (cy + ny * cz);
    cell[s] = c;
    atomicAdd(&ccount[c], 1);
  }
}

// counting-sort scatter: particle s to slot cstart[c] + rank (rank by atomic: any order inside a cell)
__global__ void k_ab_scatter(const int* __restrict__ cell, int64_t n, const int* __restrict__ cstart,
                             int* __restrict__ cfill, int* __restrict__ order) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const int c = cell[s];
    order[cstart[c] + atomicAdd(&cfill[c], 1)] = (int)s;
  }
}

// presort keys for direction d: (cell << 32) | ordered projection bits of (x - corner) . d_hat
__global__ void k_ab_keys(const float4* __restrict__ xh, const int* __restrict__ order, int64_t n,
                          const int* __restrict__ cell, int nx, int ny, float ex, float ey, float ez, int d,
                          uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int s = order[q];
    const int c = cell[s];
    const int cx = c % nx, cy = (c / nx) % ny, cz = c / (nx * ny);
    const float4 p = xh[s];
    const float3 u = dir_unit(d);
    const float key = fmaf(p.x - (float)cx * ex, u.x, fmaf(p.y - (float)cy * ey, u.y, (p.z - (float)cz * ez) * u.z));
    keys[q] = ((uint64_t)(uint32_t)c << 32) | float_ord(key);
    vals[q] = (uint32_t)s;
  }
}

struct AbParams {
  int nx, ny, nz;
  float L[3];
  const int* cstart;
  const int* ccount;
  const float4* xh;          // cell order of the build: x, y, z, h
  const float4* vm;          // v, m
  const uint32_t* sorted;    // [13][n]: per direction, particles in (cell, projection) order
  const float* proj;         // [13][n]: their projections
  const int* order;          // particles in grid-cell order (the naive loops)
  int mode;                  // 0 naive, 1 sorted
  float* rho_sum;            // [n] sum m_j f(q) (build cell order; x (8/pi) h^-3 on the host side)
  unsigned long long* ctr;   // AB_N counters
};

__device__ __forceinline__ float ab_f(float q) {   // f(q) of the cubic spline
  const float t = 1.f - q;
  return q <= 0.5f ? fmaf(q * q, fmaf(6.f, q, -6.f), 1.f) : (q < 1.f ? 2.f * t * t * t : 0.f);
}

// one warp per (cell, offset k = 13..26) pair
__global__ void __launch_bounds__(256) k_ab_pairs(AbParams P, int ncell) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= (int64_t)ncell * 14) return;
  const int ca = (int)(w / 14), k = 13 + (int)(w % 14);
  const int ax = ca % P.nx, ay = (ca / P.nx) % P.ny, az = ca / (P.nx * P.ny);
  const int ox = off_x(k), oy = off_y(k), oz = off_z(k);
  int bx = ax + ox, by = ay + oy, bz = az + oz;
  // B's periodic image is B + shift; differences are taken as (x_i - shift) - x_j, exact by
  // Sterbenz for a pair across the wrap (x_i - L for x_i near L; H2)
  float sx = 0.f, sy = 0.f, sz = 0.f;
  if (bx >= P.nx) { bx -= P.nx; sx = P.L[0]; }
  if (by >= P.ny) { by -= P.ny; sy = P.L[1]; }
  if (bz >= P.nz) { bz -= P.nz; sz = P.L[2]; }
  if (by < 0) { by += P.ny; sy = -P.L[1]; }
  if (bz < 0) { bz += P.nz; sz = -P.L[2]; }
  const int cb = bx + P.nx * (by + P.ny * bz);
  const int a0 = P.cstart[ca], na = P.ccount[ca], b0 = P.cstart[cb], nb = P.ccount[cb];
  if (na == 0 || nb == 0) return;
  const bool self = k == 13;
  const int cls = self ? 0 : dir_class(k);
  long long tests = 0, hits = 0, pass = 0, inr = 0;
  // "compute interaction" (the paper's pair update): both densities, each with its
  // own h (Eq. 2)
  auto interact = [&](int si, int sj, float r2, float hi, float hj, float& acc_i) {
    if (r2 < hi * hi) {
      acc_i = fmaf(P.vm[sj].w, ab_f(sqrtf(r2) / hi), acc_i);
      ++hits;
    }
    if (r2 < hj * hj) {
      atomicAdd(&P.rho_sum[sj], P.vm[si].w * ab_f(sqrtf(r2) / hj));
      ++hits;
    }
  };
  if (P.mode == 0 || self) {
    // naive double loop: every particle of A (lanes) against every particle of B;
    // a self pair j > i only
    for (int i0 = 0; i0 < na; i0 += 32) {
      const int ii = i0 + lane;
      const bool vi = ii < na;
      const int si = vi ? P.order[a0 + ii] : 0;
      const float4 pi = vi ? P.xh[si] : make_float4(0.f, 0.f, 0.f, 0.f);
      float acc = 0.f;
      for (int jj = self ? ii + 1 : 0; vi && jj < nb; ++jj) {
        const int sj = P.order[b0 + jj];
        const float4 pj = P.xh[sj];
        const float dx = (pi.x - sx) - pj.x, dy = (pi.y - sy) - pj.y, dz = (pi.z - sz) - pj.z;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        ++tests;
        if (!self && r2 < pi.w * pi.w) ++inr;
        if (r2 < pi.w * pi.w || r2 < pj.w * pj.w) interact(si, sj, r2, pi.w, pj.w, acc);
      }
      if (vi && acc != 0.f) atomicAdd(&P.rho_sum[si], acc);
    }
    if (!self) pass = tests;   // no window: every pair is tested
  } else {
    // sorted: A and B along the canonical direction d of offset k, projections of
    // (x - own cell corner); B's corner lies `dshift` further along d
    const int d = slot_dir(k);
    const size_t nt = (size_t)(P.cstart[ncell - 1] + P.ccount[ncell - 1]);
    const uint32_t* ls = P.sorted + (size_t)d * nt;
    const float* lp = P.proj + (size_t)d * nt;
    const float3 u = dir_unit(d);
    const float ex = P.L[0] / P.nx, ey = P.L[1] / P.ny, ez = P.L[2] / P.nz;
    const float dshift = fmaf((float)ox * ex, u.x, fmaf((float)oy * ey, u.y, (float)oz * ez * u.z));
    // sweep 1: each i of A against B in ascending projection while r_j <= r_i + h_i
    for (int i0 = 0; i0 < na; i0 += 32) {
      const int ii = i0 + lane;
      const bool vi = ii < na;
      const int si = vi ? (int)ls[a0 + ii] : 0;
      const float ri = vi ? lp[a0 + ii] : 0.f;
      const float4 pi = vi ? P.xh[si] : make_float4(0.f, 0.f, 0.f, 0.f);
      float acc = 0.f;
      for (int jj = 0; vi && jj < nb; ++jj) {
        if (ri + pi.w < lp[b0 + jj] + dshift) break;
        ++pass;
        const int sj = (int)ls[b0 + jj];
        const float4 q = P.xh[sj];
        const float dx = (pi.x - sx) - q.x, dy = (pi.y - sy) - q.y, dz = (pi.z - sz) - q.z;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        ++tests;
        if (r2 < pi.w * pi.w) {
          ++inr;
          interact(si, sj, r2, pi.w, q.w, acc);
        }
      }
      if (vi && acc != 0.f) atomicAdd(&P.rho_sum[si], acc);
    }
    // sweep 2: each j of B against A in descending projection while r_i >= r_j - h_j,
    // the pairs with r < h_j not found in sweep 1: r >= h_i (R6; the listing's r > h_i would
    // lose a pair at r == h_i exactly)
    for (int j0 = 0; j0 < nb; j0 += 32) {
      const int jj = j0 + lane;
      const bool vj = jj < nb;
      const int sj = vj ? (int)ls[b0 + jj] : 0;
      const float rj = vj ? lp[b0 + jj] + dshift : 0.f;
      const float4 q = vj ? P.xh[sj] : make_float4(0.f, 0.f, 0.f, 0.f);
      float acc = 0.f;
      for (int ii = na - 1; vj && ii >= 0; --ii) {
        if (lp[a0 + ii] < rj - q.w) break;
        const int si = (int)ls[a0 + ii];
        const float4 pi = P.xh[si];
        const float dx = (pi.x - sx) - q.x, dy = (pi.y - sy) - q.y, dz = (pi.z - sz) - q.z;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        ++tests;
        if (r2 < q.w * q.w && r2 >= pi.w * pi.w) {   // j's side only (i's h does not reach)
          acc = fmaf(P.vm[si].w, ab_f(sqrtf(r2) / q.w), acc);
          ++hits;
        }
      }
      if (vj && acc != 0.f) atomicAdd(&P.rho_sum[sj], acc);
    }
  }
  // warp totals
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tests += __shfl_xor_sync(FULL_MASK, tests, o);
    hits += __shfl_xor_sync(FULL_MASK, hits, o);
    pass += __shfl_xor_sync(FULL_MASK, pass, o);
    inr += __shfl_xor_sync(FULL_MASK, inr, o);
  }
  if (lane == 0) {
    atomicAdd(&P.ctr[AB_TESTS], (unsigned long long)tests);
    atomicAdd(&P.ctr[AB_HITS], (unsigned long long)hits);
    if (!self) {
      atomicAdd(&P.ctr[AB_PAIRS_F + cls - 1], (unsigned long long)na * (unsigned long long)nb);
      atomicAdd(&P.ctr[AB_PASS_F + cls - 1], (unsigned long long)pass);
      atomicAdd(&P.ctr[AB_INR_F + cls - 1], (unsigned long long)inr);
    }
  }
}

// the self term m_i f(0) = m_i and the sums in caller order: rho_i = (8/pi) h_i^-3 sum m f
__global__ void k_ab_finish(const uint32_t* __restrict__ perm, int64_t n, int64_t n_own, const float4* __restrict__ xh,
                            const float4* __restrict__ vm, const float* __restrict__ rho_sum, float* __restrict__ rho_out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[s];
    if (o >= n_own) continue;
    const float h = xh[s].w;
    const float hinv = 1.0f / h;
    rho_out[o] = SPH_CNORM * hinv * hinv * hinv * (rho_sum[s] + vm[s].w);
  }
}

// sorted (cell << 32 | ordered projection) keys -> particle list and projections of direction d
__global__ void k_ab_unpack(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                            uint32_t* __restrict__ ls, float* __restrict__ lp) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = (uint32_t)keys[q];
    const uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;   // inverse of float_ord
    ls[q] = vals[q];
    lp[q] = __uint_as_float(b);
  }
}
