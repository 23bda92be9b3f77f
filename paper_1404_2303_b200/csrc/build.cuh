// build.cuh — the cell hierarchy on the device (section 3.2).
//
//  a1  k_hrange                 : h0 checks, max/min h; x checks in k_keys
//  a2  k_keys                   : key = top-cell index | Morton octants to `depth` levels,
//                                 and the radix histograms; one radix sort (radix_sort.cuh)
//                                 orders every level at once (particles of a cell
//                                 contiguous in memory)
//  a3  k_pack                   : particles copied into cell order (float4 {x, y, z, h})
//  a4  k_build_levels           : recursive split of a cell into its 8 octants while
//                                 it holds "more than some minimal number" of particles and
//                                 "a reasonable fraction" of them has h < edge/2
//                                 (constants P:1354-1356); one level per launch.
//                                 split_fraction = 0 splits on the count alone.
//  a6  k_sort_leaf_warp / k_sort_leaf_block : a leaf's particles presorted along the 13
//                                 canonical pair directions, keys = projection of
//                                 (x - cell corner) on the direction; used by the sorted
//                                 sweeps of the list builder (lists.cuh).
//      k_guess_h                : initial h from cell occupancy (cold start)
//      k_leaf_groups            : targets in groups of <= 32 particles of one leaf (a warp each)
#pragma once
#include "common.cuh"

struct NodeArrays {
  int* first;       // first particle (cell order)
  int* count;
  int4* ijk;        // integer cell coordinates at its level, .w = level
  int* parent;
  int* child;       // [8*node + octant], -1 if empty / leaf
  int* split;       // 1 if split into children
  float* hmax;      // max h in the cell (force reach of the sources it holds)
  int4* rec;        // packed {first, count, first child, mask | level << 8} (k_node_rec)
  int64_t* sortoff; // offset of the node's 13 sorted lists in the sorted-entry array, -1 if none
};

struct LevelGeom {           // per-level edges (fp32), up to SPH_MAX_DEPTH+1 levels
  float E[SPH_MAX_DEPTH + 2][3];
  float L[3];
  int ntop[3];
  int depth;
};

__host__ __device__ __forceinline__ float node_corner(int i, int l, int axis, const LevelGeom& g) {
  return (float)((double)i * (double)g.E[l][axis]);
}

// ---------------------------------------------------------------- a1 ---------
// positions finite and inside [0, L) (sph_update_cells; a build validates inside k_keys)
__global__ void k_validate_x(const float* __restrict__ x, int64_t n, float Lx, float Ly, float Lz,
                             unsigned long long* ctr) {
  int err = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float a = x[3 * i], b = x[3 * i + 1], c = x[3 * i + 2];
    if (!isfinite(a) || !isfinite(b) || !isfinite(c)) err |= ERRBIT_NONFINITE;
    else if (a < 0.f || a >= Lx || b < 0.f || b >= Ly || c < 0.f || c >= Lz) err |= ERRBIT_XRANGE;
  }
  err = __reduce_or_sync(FULL_MASK, err);
  if ((threadIdx.x & 31) == 0 && err) atomicOr(&ctr[C_ERR], (unsigned long long)err);
}

// max / min positive h (float bits are monotone for h >= 0), zeros counted in C_TMP0
__global__ void k_hrange(const float* __restrict__ h, int64_t n, unsigned long long* ctr) {
  unsigned mx = 0u, mn = 0x7f800000u;
  int err = 0, zeros = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = h[i];
    if (!isfinite(v) || v < 0.f) err |= ERRBIT_H;
    else if (v > 0.f) {
      unsigned b = __float_as_uint(v);
      mx = max(mx, b);
      mn = min(mn, b);
    } else {
      ++zeros;
    }
  }
  mx = __reduce_max_sync(FULL_MASK, mx);
  mn = __reduce_min_sync(FULL_MASK, mn);
  err = __reduce_or_sync(FULL_MASK, err);
  zeros = warp_sum_i(zeros);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&ctr[C_HMAXBITS], (unsigned long long)mx);
    atomicMin(&ctr[C_HMINBITS], (unsigned long long)mn);
    if (err) atomicOr(&ctr[C_ERR], (unsigned long long)err);
    if (zeros) atomicAdd(&ctr[C_TMP0], (unsigned long long)zeros);
  }
}

// ---------------------------------------------------------------- a2 ---------
// bits of v (< 2^21) to every third bit (bit b -> bit 3b): the Morton interleave
__device__ __forceinline__ uint64_t spread3(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

// One pass over the caller's positions (a1 + a2): validation (finite, inside [0, L)), the
// cell key = top-cell index | Morton octants to `depth` levels, binned in fp64 (R19):
// cell index floor(x * n_l / L) at the deepest level, clamped; the (key, index) pairs; the
// positions packed as float4 {x, y, z, h0} in caller order (so the permute gathers one
// 16-byte record per particle); and every radix pass's digit histogram (shared-memory
// counts, one global add per block and digit).
__global__ void __launch_bounds__(256) k_keys(const float* __restrict__ x, const float* __restrict__ h0, int64_t n,
                                              float Lx, float Ly, float Lz, int nx, int ny, int nz, int depth, double sx,
                                              double sy, double sz, int npass, uint64_t* __restrict__ keys,
                                              uint32_t* __restrict__ vals, float4* __restrict__ xc,
                                              uint32_t* __restrict__ hist, unsigned long long* ctr) {
  __shared__ uint32_t sh[8][256];
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  int err = 0;
  const int64_t fx = ((int64_t)nx << depth) - 1, fy = ((int64_t)ny << depth) - 1, fz = ((int64_t)nz << depth) - 1;
  const uint64_t lowm = (1ull << depth) - 1ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float a = x[3 * i], b = x[3 * i + 1], c = x[3 * i + 2];
    if (!isfinite(a) || !isfinite(b) || !isfinite(c)) err |= ERRBIT_NONFINITE;
    else if (a < 0.f || a >= Lx || b < 0.f || b >= Ly || c < 0.f || c >= Lz) err |= ERRBIT_XRANGE;
    int64_t cx = (int64_t)floor((double)a * sx);
    int64_t cy = (int64_t)floor((double)b * sy);
    int64_t cz = (int64_t)floor((double)c * sz);
    cx = min(max(cx, (int64_t)0), fx);
    cy = min(max(cy, (int64_t)0), fy);
    cz = min(max(cz, (int64_t)0), fz);
    const uint64_t t = (uint64_t)((cx >> depth) + (int64_t)nx * ((cy >> depth) + (int64_t)ny * (cz >> depth)));
    const uint64_t m = (spread3((uint64_t)cx & lowm) << 2) | (spread3((uint64_t)cy & lowm) << 1) |
                       spread3((uint64_t)cz & lowm);
    const uint64_t k = (t << (3 * depth)) | m;
    keys[i] = k;
    vals[i] = (uint32_t)i;
    xc[i] = make_float4(a, b, c, h0 ? h0[i] : 0.f);
    for (int p = 0; p < npass; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
  }
  err = __reduce_or_sync(FULL_MASK, err);
  if ((threadIdx.x & 31) == 0 && err) atomicOr(&ctr[C_ERR], (unsigned long long)err);
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
    const uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

// ---------------------------------------------------------------- a3 ---------
// cell-order positions (and the pseudo-Verlet reference) from the packed caller-order records
__global__ void k_pack(const uint32_t* __restrict__ perm, int64_t n, const float4* __restrict__ xc,
                       float4* __restrict__ xh) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x)
    xh[s] = xc[perm[s]];
}

// top-level nodes = runs of equal top-cell index in the sorted keys
__global__ void k_mark_top(const uint64_t* __restrict__ keys, int64_t n, int sh, int* __restrict__ flag) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x)
    flag[s] = (s == 0 || (keys[s] >> sh) != (keys[s - 1] >> sh)) ? 1 : 0;
}

__global__ void k_write_top(const uint64_t* __restrict__ keys, int64_t n, int sh, const int* __restrict__ flag,
                            const int* __restrict__ idx, int nx, int ny, NodeArrays N,
                            int* __restrict__ topmap) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[s]) continue;
    int node = idx[s];
    uint64_t t = keys[s] >> sh;
    int tx = (int)(t % nx), ty = (int)((t / nx) % ny), tz = (int)(t / ((uint64_t)nx * ny));
    N.first[node] = (int)s;
    N.ijk[node] = make_int4(tx, ty, tz, 0);
    N.parent[node] = -1;
    topmap[t] = node;
  }
}

// n0 (the occupied top cells) read on the device: the grid is launched for an upper bound
__global__ void k_top_counts(const int* __restrict__ n0p, int64_t n, NodeArrays N) {
  const int n0 = *n0p;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n0) N.count[i] = (i + 1 < n0 ? N.first[i + 1] : (int)n) - N.first[i];
}

// ---------------------------------------------------------------- a4 ---------
#define GUESS_MIN_COUNT 8   // a cell counts for the occupancy guess from this many particles

// ---- a4 in one launch: every level of the hierarchy without a host round trip ------------
// A cooperative (co-resident) grid runs the level loop on the device: per level, (A) warp per
// node: split decision and octant boundaries (binary search on the keys' octant bits); (B) per-block sums of the
// children counts; (C) each block's exclusive offset from the block sums, the scan of its
// contiguous chunk of nodes and their children written. Node numbering: level by level,
// children in parent order, octant order. A level
// that would exceed the node capacity stops the loop (status[1] = 1: the host grows the
// arrays and runs it again).
#ifndef SORT_BLOCK_MAX
#define SORT_BLOCK_MAX 4096
#endif
struct LevelBuild {
  int* lev_off;      // [SPH_MAX_DEPTH + 4]: level offsets (zeroed by the host; [1] = n0 written here)
  int* status;       // [0] levels processed, [1] 1 = node capacity exceeded, 2 = barrier timeout
  unsigned* bar;     // grid barrier: arrivals, generation (zeroed before the launch)
  int* part;         // [gridDim.x] block sums
  int* nch;          // [cap] children per node of the level being built (index node - a)
  int cap;           // node capacity
  int* presort;      // set to 1 if a leaf qualifies for presorted lists (count > sort_min_len): the
                     // host skips the presort pass (and its scan's round trip) when it stays 0
  int sort_min_len;
  int* ngroups;      // target groups of the tree (cmax > 0: chunks of <= SPH_GROUP of every container,
  int cmax;          // as k_group_count counts them), summed here so the host needs no scan total
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// all blocks of a co-resident grid meet here; false if the wait timed out (a stalled grid
// exits with an error instead of hanging the device)
__device__ __forceinline__ bool grid_sync(unsigned* bar, int* status) {
  __shared__ int ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    ok = 1;
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const unsigned long long t0 = globaltimer_ns();
      while (*gen == g) {
        __nanosleep(100);
        if (globaltimer_ns() - t0 > 2000000000ull) {
          ok = 0;
          atomicExch(status + 1, 2);
          break;
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
  return ok;
}

__device__ __forceinline__ int block_sum_i(int v, int* red) {
  v = warp_sum_i(v);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  int t = 0;
  for (int k = 0; k < nw; ++k) t += red[k];
  return t;
}

#define LEVEL_THREADS 256
#ifndef LEVEL_CHUNK_A
#define LEVEL_CHUNK_A 1   // phase A over the block's own chunk of nodes: one grid barrier per level fewer (C4 -0.02 ms)
#endif
// guess_n > 0: a cold start; each leaf, once decided, writes the occupancy guess of h (as
// k_guess_h, n_ngb = guess_n, ancestors up to |guess_min| particles) into xh_w[].w where 0
// (guess_min < 0: into every particle's, no h0 was given).
__global__ void __launch_bounds__(LEVEL_THREADS) k_build_levels(LevelBuild L, const float4* __restrict__ xh,
                                                                const uint64_t* __restrict__ keys, LevelGeom g,
                                                                int depth, int split_count, float split_frac,
                                                                NodeArrays N, float guess_n, int guess_min,
                                                                float hcap, float4* xh_w, const int* n0p) {
  const int n0 = __ldcg(n0p);   // the occupied top cells (a device scan total: no host round trip)
  __shared__ int red[LEVEL_THREADS / 32];
  __shared__ int wsc[LEVEL_THREADS / 32];
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(gridDim.x * (blockDim.x >> 5));
  volatile int* lev = L.lev_off;
  int wgroups = 0;   // lane 0: groups of the containers this warp decided (all levels)
  for (int l = 0;; ++l) {
    // level 0 (the top cells, 0..n0) from the argument: lev[] is written only under barriers
    const int a = l == 0 ? 0 : lev[l], b = l == 0 ? n0 : lev[l + 1];
    const float half_edge = 0.5f * fminf(g.E[l][0], fminf(g.E[l][1], g.E[l][2]));
    // the block's contiguous chunk of the level (phase B sums it, phase C writes its children)
    const int nl = b - a;
    const int chunk = (nl + gridDim.x - 1) / gridDim.x;
    const int c0 = a + min(nl, (int)blockIdx.x * chunk), c1 = a + min(nl, ((int)blockIdx.x + 1) * chunk);
    // (A) split decision + octant boundaries, warp per node
#if LEVEL_CHUNK_A
    // over the block's own chunk: (B) then follows without a grid barrier
    for (int node = c0 + (int)(threadIdx.x >> 5); node < c1; node += (int)(blockDim.x >> 5)) {
#else
    for (int node = a + gw; node < b; node += nwarps) {
#endif
      const int first = __ldcg(N.first + node), cnt = __ldcg(N.count + node);
      bool frac_ok = true;
      if (split_frac > 0.f && cnt > split_count && l < depth) {
        int nsmall = 0;
        for (int s = first + lane; s < first + cnt; s += 32) nsmall += (xh[s].w < half_edge) ? 1 : 0;
        nsmall = warp_sum_i(nsmall);
        frac_ok = (double)nsmall > (double)split_frac * (double)cnt;
      }
      const int sp = (l < depth) && (cnt > split_count) && frac_ok;
      if (lane == 0) N.split[node] = sp;
      if (lane == 0 && L.cmax > 0) {   // is_container (below), with this level's split decision
        const int par = __ldcg(N.parent + node);
        const bool cont = cnt <= L.cmax ? (par < 0 || __ldcg(N.count + par) > L.cmax) : !sp;
        if (cont) wgroups += (cnt + SPH_GROUP - 1) / SPH_GROUP;
      }
      if (lane == 0 && !sp && cnt > L.sort_min_len && cnt > 1 && cnt <= SORT_BLOCK_MAX) *L.presort = 1;
      if (!sp) {
        if (lane == 0) L.nch[node - a] = 0;
        if (guess_n > 0.f) {
          float dens = 0.f;
          int y = node;
          while (true) {
            const int cy = __ldcg(N.count + y);
            const int ly = __ldcg(N.ijk + y).w;
            const float vol = g.E[ly][0] * g.E[ly][1] * g.E[ly][2];
            if (cy >= GUESS_MIN_COUNT) dens = fmaxf(dens, (float)cy / vol);
            const int py = __ldcg(N.parent + y);
            if (cy >= abs(guess_min) || py < 0) {
              if (dens == 0.f) dens = (float)cy / vol;
              break;
            }
            y = py;
          }
          const float hg = fminf(cbrtf(3.f * guess_n / (4.f * 3.14159265f * dens)), hcap);
          if (guess_min < 0) {   // no h0 at all: every particle takes the guess (no read)
            for (int s = first + lane; s < first + cnt; s += 32) xh_w[s].w = hg;
          } else {
            for (int s = first + lane; s < first + cnt; s += 32)
              if (xh_w[s].w == 0.f) xh_w[s].w = hg;
          }
        }
        continue;
      }
      // octant boundaries: a binary search per octant on the sorted keys (lanes 0..7)
      const int shift = 3 * (depth - l - 1);
      int start = first + cnt;
      if (lane < 8) {
        int lo = first, hi = first + cnt;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const int oct = (int)((keys[mid] >> shift) & 7ull);
          if (oct < lane) lo = mid + 1;
          else hi = mid;
        }
        start = lo;
      }
      const int nxt = __shfl_down_sync(FULL_MASK, start, 1);
      const unsigned bal = __ballot_sync(FULL_MASK, lane < 8 && nxt - start > 0);
      if (lane < 8) N.child[8 * (int64_t)node + lane] = start;
      if (lane == 0) L.nch[node - a] = __popc(bal);
    }
    if (lane == 0 && wgroups) {
      atomicAdd(L.ngroups, wgroups);
      wgroups = 0;
    }
#if LEVEL_CHUNK_A
    __syncthreads();   // the block's nch entries are its own writes
#else
    if (!grid_sync(L.bar, L.status)) return;
#endif
    // (B) block sums over contiguous chunks of the level
    int v = 0;
    for (int p = c0 + threadIdx.x; p < c1; p += blockDim.x) v += __ldcg(L.nch + (p - a));
    v = block_sum_i(v, red);
    if (threadIdx.x == 0) L.part[blockIdx.x] = v;
    if (!grid_sync(L.bar, L.status)) return;
    // (C) offsets, scan of the chunk, children
    int before = 0, total = 0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
      const int pk = __ldcg(L.part + k);
      total += pk;
      if (k < (int)blockIdx.x) before += pk;
    }
    before = block_sum_i(before, red);
    total = block_sum_i(total, red);
    const int next = b + total;
    if (next > L.cap) {   // the same decision in every block: no block waits at a barrier below
      if (blockIdx.x == 0 && threadIdx.x == 0) L.status[1] = 1;
      return;
    }
    int carry = b + before;
    for (int t0 = c0; t0 < c1; t0 += blockDim.x) {
      const int p = t0 + threadIdx.x;
      const int nc = p < c1 ? __ldcg(L.nch + (p - a)) : 0;
      // block exclusive scan of nc
      int incl = nc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o) incl += y;
      }
      __syncthreads();
      if (lane == 31) wsc[threadIdx.x >> 5] = incl;
      __syncthreads();
      int wpre = 0, ttot = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
        if (k < (int)(threadIdx.x >> 5)) wpre += wsc[k];
        ttot += wsc[k];
      }
      if (p < c1) {
        int* ch = N.child + 8 * (int64_t)p;
        if (nc == 0) {
#pragma unroll
          for (int o = 0; o < 8; ++o) ch[o] = -1;
        } else {
          int st[9];
#pragma unroll
          for (int o = 0; o < 8; ++o) st[o] = __ldcg(ch + o);
          st[8] = __ldcg(N.first + p) + __ldcg(N.count + p);
          const int4 pijk = __ldcg(N.ijk + p);
          const int base = carry + wpre + incl - nc;
          int k = 0;
#pragma unroll
          for (int o = 0; o < 8; ++o) {
            const int cc = st[o + 1] - st[o];
            if (cc > 0) {
              const int cn = base + k++;
              N.first[cn] = st[o];
              N.count[cn] = cc;
              N.ijk[cn] = make_int4(2 * pijk.x + ((o >> 2) & 1), 2 * pijk.y + ((o >> 1) & 1), 2 * pijk.z + (o & 1),
                                    pijk.w + 1);
              N.parent[cn] = p;
              ch[o] = cn;
            } else {
              ch[o] = -1;
            }
          }
        }
      }
      carry += ttot;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (l == 0) L.lev_off[1] = n0;
      L.lev_off[l + 2] = next;
      L.status[0] = l + 1;
    }
    if (total == 0) return;
    if (!grid_sync(L.bar, L.status)) return;
  }
}

// per node max of a per-particle value (cell order), warp per node
// (values >= 0); the top cells' maxima also give the global max (ctr[C_HMAXBITS], if set)
__global__ void k_node_hmax(int nnodes, NodeArrays N, const float* __restrict__ h, unsigned long long* ctr) {
  const int lane = threadIdx.x & 31;
  const int node = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= nnodes) return;
  const int first = N.first[node], cnt = N.count[node];
  float hm = 0.f;
  for (int s = first + lane; s < first + cnt; s += 32) hm = fmaxf(hm, h[s]);
  hm = warp_max_f(hm);
  if (lane == 0) {
    N.hmax[node] = hm;
    if (ctr && N.parent[node] < 0) atomicMax(&ctr[C_HMAXBITS], (unsigned long long)__float_as_uint(hm));
  }
}

// initial guess from cell occupancy: N = (4 pi/3) n h^3 for a uniform number density n
// (Eq. 3) -> h = cbrt(3 N_ngb / (4 pi n)). n is the largest number density among the leaf
// and its ancestors holding >= GUESS_MIN_COUNT particles, up to the first ancestor holding
// >= n_ngb: next to a dense clump a sparse cell's mean density hides the clump, and an
// over-estimated h costs a long interaction list while an under-estimate costs one Newton
// step. Written in cell order into xh[].w where h == 0.
__global__ void k_guess_h(int nnodes, NodeArrays N, LevelGeom g, float n_ngb, int min_count, float hcap,
                          float4* __restrict__ xh) {
  const int lane = threadIdx.x & 31;
  const int x = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (x >= nnodes || N.split[x]) return;
  double dens = 0.0;
  int y = x;
  while (true) {
    const int cnt = N.count[y];
    const int l = N.ijk[y].w;
    if (cnt >= GUESS_MIN_COUNT) {
      const double vol = (double)g.E[l][0] * g.E[l][1] * g.E[l][2];
      dens = fmax(dens, (double)cnt / vol);
    }
    if (cnt >= min_count || N.parent[y] < 0) {
      if (dens == 0.0) dens = (double)cnt / ((double)g.E[l][0] * g.E[l][1] * g.E[l][2]);
      break;
    }
    y = N.parent[y];
  }
  float h = (float)cbrt(3.0 * n_ngb / (4.0 * 3.14159265358979323846 * dens));
  h = fminf(h, hcap);
  for (int s = N.first[x] + lane; s < N.first[x] + N.count[x]; s += 32)
    if (xh[s].w == 0.f) xh[s].w = h;
}

// packed node records for the list walk: {first, count, first child (-1: none),
// octant mask of the children | level << 8}; children are allocated contiguously in
// octant order by k_build_levels
__global__ void k_node_rec(int nnodes, NodeArrays N, int4* __restrict__ rec) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  int base = -1, mask = 0;
  if (N.split[x]) {
    for (int o = 0; o < 8; ++o) {
      const int ch = N.child[8 * (int64_t)x + o];
      if (ch >= 0) {
        if (base < 0) base = ch;
        mask |= 1 << o;
      }
    }
  }
  rec[x] = make_int4(N.first[x], N.count[x], base, mask | (N.ijk[x].w << 8));
}

// ---------------------------------------------------------------- a6 ---------
__device__ __forceinline__ float proj(float rx, float ry, float rz, float3 d) {
  return fmaf(rx, d.x, fmaf(ry, d.y, rz * d.z));
}

struct SortEntry {  // 8 bytes: projection key and cell-order particle index
  float key;
  int idx;
};

// number of sorted entries of each leaf: 13 * count if it is presorted
__global__ void k_sort_sizes(int nnodes, NodeArrays N, int sort_min_len, int64_t* __restrict__ sz) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= nnodes) return;
  const int cnt = N.count[y];
  const bool srt = !N.split[y] && cnt > sort_min_len && cnt <= SORT_BLOCK_MAX && cnt > 1;
  sz[y] = srt ? 13 * (int64_t)cnt : 0;
}
__global__ void k_sort_offsets(int nnodes, const int64_t* __restrict__ sz, const int64_t* __restrict__ scan,
                               NodeArrays N) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= nnodes) return;
  N.sortoff[y] = sz[y] > 0 ? scan[y] : -1;
}

// warp per leaf with count <= 32: warp bitonic sort of (key, lane) per direction
__global__ void k_sort_leaf_warp(int nnodes, const float4* __restrict__ xh, NodeArrays N, LevelGeom g,
                                 SortEntry* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int node = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= nnodes) return;
  const int64_t off = N.sortoff[node];
  const int cnt = N.count[node];
  if (off < 0 || cnt > 32) return;
  const int first = N.first[node];
  const int4 c = N.ijk[node];
  float rx = 0.f, ry = 0.f, rz = 0.f;
  if (lane < cnt) {
    float4 p = xh[first + lane];
    rx = p.x - node_corner(c.x, c.w, 0, g);
    ry = p.y - node_corner(c.y, c.w, 1, g);
    rz = p.z - node_corner(c.z, c.w, 2, g);
  }
  for (int d = 0; d < 13; ++d) {
    const float key = proj(rx, ry, rz, dir_unit(d));
    uint64_t v = lane < cnt ? (((uint64_t)float_ord(key) << 32) | (uint32_t)lane) : ~0ull;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        uint64_t o = __shfl_xor_sync(FULL_MASK, v, stride);
        bool up = ((lane & size) == 0);
        bool lower = ((lane & stride) == 0);
        uint64_t mn = v < o ? v : o, mx = v < o ? o : v;
        v = (lower == up) ? mn : mx;
      }
    }
    const int li = (lane < cnt) ? (int)(uint32_t)v : 0;
    const float kk = __shfl_sync(FULL_MASK, key, li);
    if (lane < cnt) out[off + (int64_t)d * cnt + lane] = SortEntry{kk, first + li};
  }
}

// CTA per leaf with 32 < count <= SORT_BLOCK_MAX: shared-memory bitonic sort per direction
__global__ void __launch_bounds__(512) k_sort_leaf_block(int nnodes, const float4* __restrict__ xh, NodeArrays N,
                                                         LevelGeom g, SortEntry* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sb_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(sb_raw);
  float* skey = reinterpret_cast<float*>(sk + SORT_BLOCK_MAX);
  const int node = blockIdx.x;
  if (node >= nnodes) return;
  const int64_t off = N.sortoff[node];
  const int cnt = N.count[node];
  if (off < 0 || cnt <= 32) return;
  const int first = N.first[node];
  const int4 c = N.ijk[node];
  const float cx = node_corner(c.x, c.w, 0, g), cy = node_corner(c.y, c.w, 1, g), cz = node_corner(c.z, c.w, 2, g);
  int P = 64;
  while (P < cnt) P <<= 1;
  for (int d = 0; d < 13; ++d) {
    const float3 dv = dir_unit(d);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < cnt) {
        const float4 p = xh[first + i];
        const float key = proj(p.x - cx, p.y - cy, p.z - cz, dv);
        skey[i] = key;
        sk[i] = ((uint64_t)float_ord(key) << 32) | (uint32_t)i;
      } else {
        sk[i] = ~0ull;
      }
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool up = ((lo & size) == 0);
          const uint64_t A = sk[lo], B = sk[hi];
          if ((A > B) == up) {
            sk[lo] = B;
            sk[hi] = A;
          }
        }
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const int li = (int)(uint32_t)sk[i];
      out[off + (int64_t)d * cnt + i] = SortEntry{skey[li], first + li};
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- groups -----
// Targets in groups of <= SPH_GROUP particles (one warp each in the interaction kernels),
// each a contiguous range of the cell order that lies inside one cell:
//   * the children of a split cell that are leaves are packed greedily, in octant order,
//     into runs of consecutive siblings holding <= SPH_GROUP particles (consecutive
//     siblings are contiguous in memory, and they all lie inside the parent's box);
//   * a leaf with more than SPH_GROUP particles (the paper's split rule keeps leaves of
//     up to split_count particles; coincident particles at the deepest level) is cut into
//     balanced chunks of consecutive particles (Morton order inside the leaf);
//   * a top-level leaf is its own group.
// int4 {node, first, count, -}.
__device__ __forceinline__ int n_chunks(int cnt) { return (cnt + SPH_GROUP - 1) / SPH_GROUP; }

template <bool WRITE>
__device__ __forceinline__ int pack_children(const NodeArrays& N, int x, int4* out) {
  int g = 0, acc = 0, first = 0;
  for (int o = 0; o < 8; ++o) {
    const int ch = N.child[8 * (int64_t)x + o];
    if (ch < 0) continue;
    const int cnt = N.count[ch];
    if (N.split[ch] || cnt > SPH_GROUP) {            // handled at its own node
      if (acc > 0) {
        if (WRITE) out[g] = make_int4(x, first, acc, 0);
        ++g;
        acc = 0;
      }
      continue;
    }
    if (acc + cnt > SPH_GROUP) {
      if (WRITE) out[g] = make_int4(x, first, acc, 0);
      ++g;
      acc = 0;
    }
    if (acc == 0) first = N.first[ch];
    acc += cnt;
  }
  if (acc > 0) {
    if (WRITE) out[g] = make_int4(x, first, acc, 0);
    ++g;
  }
  return g;
}

// With cmax > 0 a group container is the deepest cell holding <= cmax particles (or a leaf
// holding more): its particles, contiguous in Morton order, are cut into balanced chunks.
__device__ __forceinline__ bool is_container(const NodeArrays& N, int x, int cmax) {
  const int cnt = N.count[x];
  if (cnt <= cmax) return N.parent[x] < 0 || N.count[N.parent[x]] > cmax;
  return !N.split[x];
}

__global__ void k_group_count(int nnodes, NodeArrays N, int cmax, int* __restrict__ ng) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  const int cnt = N.count[x];
  int g = 0;
  if (cmax > 0) g = is_container(N, x, cmax) ? n_chunks(cnt) : 0;
  else if (N.split[x]) g = pack_children<false>(N, x, nullptr);
  else if (N.parent[x] < 0 || cnt > SPH_GROUP) g = n_chunks(cnt);
  ng[x] = g;
}

__global__ void k_group_write(int nnodes, NodeArrays N, int cmax, const int* __restrict__ scan,
                              int4* __restrict__ groups) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  const int cnt = N.count[x], first = N.first[x];
  int4* out = groups + scan[x];
  if (cmax > 0 ? !is_container(N, x, cmax) : false) return;
  if (cmax <= 0 && N.split[x]) {
    pack_children<true>(N, x, out);
  } else if (cmax > 0 || N.parent[x] < 0 || cnt > SPH_GROUP) {
    const int c = n_chunks(cnt);
    for (int i = 0; i < c; ++i) {      // balanced: 40 -> 20 + 20
      const int s0 = (int)((int64_t)cnt * i / c), s1 = (int)((int64_t)cnt * (i + 1) / c);
      out[i] = make_int4(x, first + s0, s1 - s0, 0);
    }
  }
}

// Pseudo-Verlet reuse of the cells: the new positions of the same particles
// in the cell order of the last full build, each kept as ref + its minimum-image
// displacement (so it stays next to the cell it was sorted into, even across the periodic
// boundary), h from h_in; the largest displacement component into ctr[C_HMAXBITS].
__global__ void k_update_pos(const uint32_t* __restrict__ perm, int64_t n, const float* __restrict__ x_in,
                             const float* __restrict__ h_in, const float4* __restrict__ xref, float Lx, float Ly,
                             float Lz, float4* __restrict__ xh, unsigned long long* ctr) {
  unsigned mx = 0u;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = perm[s];
    const float4 r = xref[s];
    const float L[3] = {Lx, Ly, Lz};
    const float xn[3] = {x_in[3 * (int64_t)o], x_in[3 * (int64_t)o + 1], x_in[3 * (int64_t)o + 2]};
    const float rr[3] = {r.x, r.y, r.z};
    float y[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      float d = xn[k] - rr[k];
      if (d > 0.5f * L[k]) d -= L[k];
      if (d < -0.5f * L[k]) d += L[k];
      y[k] = rr[k] + d;
      mx = max(mx, __float_as_uint(fabsf(d)));
    }
    xh[s] = make_float4(y[0], y[1], y[2], h_in[o]);
  }
  mx = __reduce_max_sync(FULL_MASK, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(&ctr[C_HMAXBITS], (unsigned long long)mx);
}
