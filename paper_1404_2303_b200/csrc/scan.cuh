// scan.cuh — exclusive prefix sums (int32 / int64) used for compactions and offsets.
// Three launches: per-block totals, a single-block scan of the totals, per-block scan
// plus carry. Blocks of 1024 threads x 4 items.
#pragma once
#include "common.cuh"

#define SCAN_THREADS 1024
#define SCAN_ITEMS 4
#define SCAN_TILE (SCAN_THREADS * SCAN_ITEMS)

template <typename T>
__device__ __forceinline__ T block_incl_scan(T x, T* smem_w /*[32]*/, T* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(FULL_MASK, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_w[w] = x;
  __syncthreads();
  if (w == 0) {
    T s = (lane < (int)(blockDim.x >> 5)) ? smem_w[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(FULL_MASK, s, o);
      if (lane >= o) s += y;
    }
    smem_w[lane] = s;
  }
  __syncthreads();
  T add = (w > 0) ? smem_w[w - 1] : T(0);
  if (total) *total = smem_w[(blockDim.x >> 5) - 1];
  return x + add;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const T* __restrict__ in, int64_t n,
                                                              T* __restrict__ block_sums) {
  __shared__ T sw[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i)
    if (base + i < n) s += in[base + i];
  T tot;
  block_incl_scan<T>(s, sw, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_blocksums(T* __restrict__ sums, int64_t nb,
                                                                 T* __restrict__ total_out) {
  __shared__ T sw[32];
  __shared__ T carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += SCAN_THREADS) {
    int64_t i = b0 + threadIdx.x;
    T x = (i < nb) ? sums[i] : T(0);
    T tot;
    T inc = block_incl_scan<T>(x, sw, &tot);
    T c = carry;
    if (i < nb) sums[i] = c + inc - x;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_final(const T* __restrict__ in, int64_t n,
                                                             const T* __restrict__ block_sums,
                                                             T* __restrict__ out) {
  __shared__ T sw[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  T v[SCAN_ITEMS];
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = (base + i < n) ? in[base + i] : T(0);
    s += v[i];
  }
  T inc = block_incl_scan<T>(s, sw, nullptr);
  T run = inc - s + block_sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
}
