// radix_sort.cuh — hand-written LSD radix sort of (u64 key, u32 value) pairs for sm_100a.
//
// Onesweep structure: one histogram kernel computes every pass's digit counts in a
// single read of the keys (fused into k_keys, build.cuh); each 8-bit pass is then ONE
// kernel: tiles of 2048 items
// ranked in-warp from digit-bit ballots (stable), tile digit counts published with a
// decoupled look-back (per-digit status words), items staged in shared memory in
// digit order and written out in coalesced digit runs. Digit offsets are scanned on the
// device (k_radix_offsets); every pass runs, so the sort has no host round trip.
#pragma once
#include "common.cuh"

#ifndef RS_THREADS
#define RS_THREADS 512  // 256 or 512 (the first 256 threads hold one digit each in the scan / look-back);
                        // 4096-item tiles halve the tiles in flight a look-back walks over (16.8M: -2.4%)
#endif
#ifndef RS_ITEMS
#define RS_ITEMS 8      // 8 items per thread: <= 64 registers, 1024 threads per SM (16 items: 128 registers,
#endif                  // 2 blocks, +36% on the 16.8M binning run; profiles/round2/binning_*.txt)
#define RS_TILE (RS_THREADS * RS_ITEMS)
#ifndef RS_LB
#define RS_LB 8         // predecessor statuses loaded together in the look-back
#endif
#define RS_WARPS (RS_THREADS / 32)
#define RS_FLAG_INC 0x80000000u
#define RS_FLAG_AGG 0x40000000u
#define RS_VAL_MASK 0x3fffffffu

__global__ void __launch_bounds__(256) k_radix_hist(const uint64_t* __restrict__ keys, int64_t n,
                                                     int npass, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    for (int p = 0; p < npass; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// exclusive prefix of each pass's 256 digit counts (block p = pass p): the global digit
// offsets, computed on the device so the sort needs no host round trip
__global__ void __launch_bounds__(256) k_radix_offsets(const uint32_t* __restrict__ hist, uint32_t* __restrict__ gofs) {
  __shared__ uint32_t s[256];
  const int p = blockIdx.x, d = threadIdx.x;
  const uint32_t v = hist[p * 256 + d];
  s[d] = v;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const uint32_t y = d >= o ? s[d - o] : 0u;
    __syncthreads();
    s[d] += y;
    __syncthreads();
  }
  gofs[p * 256 + d] = s[d] - v;
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

struct RadixSmem {
  uint32_t wcnt[RS_WARPS][256];
  uint32_t dpre[256];
  uint32_t gbase[256];
  uint32_t tile;
  uint32_t wsum[RS_WARPS];
  uint64_t keys[RS_TILE];
  uint32_t vals[RS_TILE];
};

#ifndef RS_MINB
#define RS_MINB (1024 / RS_THREADS)   // 64 registers: 1024 resident threads per SM
#endif
__global__ void __launch_bounds__(RS_THREADS, RS_MINB) k_radix_pass(
    const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n, int shift, const uint32_t* __restrict__ gofs,
    uint32_t* status, uint32_t* tile_ctr) {
  extern __shared__ __align__(16) unsigned char rs_raw[];
  RadixSmem& S = *reinterpret_cast<RadixSmem*>(rs_raw);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int i = tid; i < RS_WARPS * 256; i += RS_THREADS) (&S.wcnt[0][0])[i] = 0;
  if (tid == 0) S.tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = S.tile;
  const int64_t base = (int64_t)tile * RS_TILE;
  const int tile_n = (int)min((int64_t)RS_TILE, n - base);

  uint64_t k[RS_ITEMS];
  uint32_t v[RS_ITEMS];
  uint32_t rank[RS_ITEMS];
  uint32_t dg[RS_ITEMS];
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    int li = w * (RS_ITEMS * 32) + it * 32 + lane;
    if (li < tile_n) {
      k[it] = kin[base + li];
      v[it] = vin[base + li];
      dg[it] = (uint32_t)(k[it] >> shift) & 255u;
    } else {
      k[it] = 0;
      v[it] = 0;
      dg[it] = 256u;
    }
  }
  // stable in-warp ranking: items visited in position order (it major, lane minor); the
  // lanes holding the same digit from ballots of the 8 digit bits (+ the invalid flag in a
  // partial tile), cheaper than __match_any_sync
  const bool full = tile_n == RS_TILE;
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    uint32_t d = dg[it];
    unsigned peers = FULL_MASK;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const bool bit = (d >> b) & 1u;
      const unsigned bb = __ballot_sync(FULL_MASK, bit);
      peers &= bit ? bb : ~bb;
    }
    if (!full) {
      const bool bit = d >> 8;
      const unsigned bb = __ballot_sync(FULL_MASK, bit);
      peers &= bit ? bb : ~bb;
    }
    uint32_t cnt_before = 0;
    if (d < 256u) cnt_before = S.wcnt[w][d];
    __syncwarp();
    rank[it] = cnt_before + __popc(peers & lanemask_lt());
    if (d < 256u && lane == __ffs(peers) - 1) S.wcnt[w][d] = cnt_before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread d < 256): exclusive over warps, the tile total published at once as
  // the tile's aggregate, and the tile-local exclusive prefix over digits
  const int d = tid;
  const bool digit = tid < 256;
  uint32_t tcnt = 0, x = 0;
  uint32_t* st = status + (size_t)tile * 256 + (digit ? d : 0);
  if (digit) {
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
      uint32_t c = S.wcnt[ww][d];
      S.wcnt[ww][d] = run;
      run += c;
    }
    tcnt = run;
    if (tile == 0) {
      atomicExch(st, RS_FLAG_INC | tcnt);
      S.gbase[d] = gofs[d];
    } else {
      atomicExch(st, RS_FLAG_AGG | tcnt);
    }
    x = tcnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(FULL_MASK, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) S.wsum[w] = x;
  }
  __syncthreads();
  if (digit) {
    uint32_t add = 0;
    for (int ww = 0; ww < w; ++ww) add += S.wsum[ww];
    S.dpre[d] = x - tcnt + add;
  }
  __syncthreads();
  // the tile sorted by digit in shared memory: this work sits between the tile's aggregate
  // and its look-back, so the predecessors have mostly published their inclusive prefix by
  // the time it is read
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    uint32_t dd = dg[it];
    if (dd < 256u) {
      uint32_t pos = S.dpre[dd] + S.wcnt[w][dd] + rank[it];
      S.keys[pos] = k[it];
      S.vals[pos] = v[it];
    }
  }
  // decoupled look-back over the previous tiles for digit d: the predecessor first (usually
  // inclusive by now), then RS_LB statuses at a time
  if (digit && tile != 0) {
    uint32_t excl = 0;
    int64_t pt = (int64_t)tile - 1;
    uint32_t s0 = ld_volatile_u32(status + (size_t)pt * 256 + d);
    while ((s0 & (RS_FLAG_INC | RS_FLAG_AGG)) == 0) s0 = ld_volatile_u32(status + (size_t)pt * 256 + d);
    excl = s0 & RS_VAL_MASK;
    bool done = (s0 & RS_FLAG_INC) != 0;
    --pt;
    while (!done) {
      uint32_t sv[RS_LB];
#pragma unroll
      for (int k2 = 0; k2 < RS_LB; ++k2)
        sv[k2] = pt - k2 >= 0 ? ld_volatile_u32(status + (size_t)(pt - k2) * 256 + d) : RS_FLAG_INC;
#pragma unroll
      for (int k2 = 0; k2 < RS_LB; ++k2) {
        if (done) break;
        while ((sv[k2] & (RS_FLAG_INC | RS_FLAG_AGG)) == 0)
          sv[k2] = ld_volatile_u32(status + (size_t)(pt - k2) * 256 + d);
        excl += sv[k2] & RS_VAL_MASK;
        if (sv[k2] & RS_FLAG_INC) done = true;
      }
      pt -= RS_LB;
    }
    atomicExch(st, RS_FLAG_INC | (excl + tcnt));
    S.gbase[d] = gofs[d] + excl;
  }
  __syncthreads();
  for (int i = tid; i < tile_n; i += RS_THREADS) {
    uint64_t kk = S.keys[i];
    uint32_t dd = (uint32_t)(kk >> shift) & 255u;
    uint32_t g = S.gbase[dd] + (uint32_t)i - S.dpre[dd];
    kout[g] = kk;
    vout[g] = S.vals[i];
  }
}
