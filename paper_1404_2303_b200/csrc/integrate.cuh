// integrate.cuh — the step around the hot path (first part): velocity-Verlet
// kick and drift of the particles ("integrated using a velocity-Verlet
// integrator") and the per-particle time step of Eq. 6,
//   dt_i = C_CFL 2 h_i / max_j (c_i + c_j + max{0, -3 r_ij . v_ij / r_ij}) = C_CFL 2 h_i / vsig_i,
// with vsig from the force loop (k_force). Arrays in the caller's order, device memory.
#pragma once
#include "common.cuh"

// kick: v += a dt, u += du/dt dt
__global__ void k_kick(int64_t n, float* __restrict__ v, float* __restrict__ u, const float* __restrict__ a,
                       const float* __restrict__ dudt, float dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    v[3 * i] = fmaf(a[3 * i], dt, v[3 * i]);
    v[3 * i + 1] = fmaf(a[3 * i + 1], dt, v[3 * i + 1]);
    v[3 * i + 2] = fmaf(a[3 * i + 2], dt, v[3 * i + 2]);
    if (u) u[i] = fmaf(dudt[i], dt, u[i]);
  }
}

// kick with a per-particle step (individual time steps): v += a dt_i,
// u += du/dt dt_i; dt_i = 0 leaves a particle as it is
__global__ void k_kick_each(int64_t n, float* __restrict__ v, float* __restrict__ u, const float* __restrict__ a,
                            const float* __restrict__ dudt, const float* __restrict__ dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = dt[i];
    if (d == 0.f) continue;
    v[3 * i] = fmaf(a[3 * i], d, v[3 * i]);
    v[3 * i + 1] = fmaf(a[3 * i + 1], d, v[3 * i + 1]);
    v[3 * i + 2] = fmaf(a[3 * i + 2], d, v[3 * i + 2]);
    if (u) u[i] = fmaf(dudt[i], d, u[i]);
  }
}

// drift: x += v dt, wrapped back into [0, L) (periodic box); |v dt| < L
__device__ __forceinline__ float wrap1(float x, float L) {
  if (x >= L) x -= L;
  if (x < 0.f) x += L;
  return (x >= L || x < 0.f) ? 0.f : x;   // a rounding onto L itself lands on 0
}
__global__ void k_drift(int64_t n, float* __restrict__ x, const float* __restrict__ v, float dt, float Lx, float Ly,
                        float Lz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[3 * i] = wrap1(fmaf(v[3 * i], dt, x[3 * i]), Lx);
    x[3 * i + 1] = wrap1(fmaf(v[3 * i + 1], dt, x[3 * i + 1]), Ly);
    x[3 * i + 2] = wrap1(fmaf(v[3 * i + 2], dt, x[3 * i + 2]), Lz);
  }
}

// Eq. 6 per particle (optional output) and its minimum (float bits, atomicMin on positives)
__global__ void k_timestep(int64_t n, const float* __restrict__ h, const float* __restrict__ vsig, float c_cfl,
                           float* __restrict__ dt_out, unsigned* __restrict__ dt_min_bits) {
  unsigned mn = 0x7f800000u;   // +inf
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float dt = vsig[i] > 0.f ? c_cfl * 2.f * h[i] / vsig[i] : INFINITY;
    if (dt_out) dt_out[i] = dt;
    mn = min(mn, __float_as_uint(dt));
  }
  mn = __reduce_min_sync(FULL_MASK, mn);
  if ((threadIdx.x & 31) == 0) atomicMin(dt_min_bits, mn);
}

// Individual time steps: power-of-two step in dt_min ticks <= the Eq. 6 step,
// dividing ti, at most 2x the previous one (include/sph.h sph_timebins)
__global__ void k_timebins(int64_t n, const float* __restrict__ h, const float* __restrict__ vsig, float c_cfl,
                           double dt_min, int n_bins, long long ti, const uint8_t* __restrict__ active,
                           const long long* __restrict__ tin, int cap2, long long* __restrict__ tout) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (active && !active[i]) {
      tout[i] = tin ? tin[i] : 1;
      continue;
    }
    const double dt = vsig[i] > 0.f ? (double)(c_cfl * 2.f * h[i] / vsig[i]) : INFINITY;
    const double q = fmax(dt / dt_min, 1.0);
    int k = q >= (double)(1ll << n_bins) ? n_bins : (int)floor(log2(q));
    k = min(max(k, 0), n_bins);
    long long s = 1ll << k;
    while (s > 1 && ti % s != 0) s >>= 1;                         // on its own grid
    if (tin && cap2) s = min(s, 2 * tin[i]);                       // grows at most 2x
    tout[i] = s;
  }
}

// limiter wake-up (include/sph.h sph_timebins_wake)
__global__ void k_timebins_wake(int64_t n, const uint8_t* __restrict__ active, const float* __restrict__ lim,
                                long long ti_end, const long long* __restrict__ begin, long long* __restrict__ ticks,
                                double dt_min, float* __restrict__ kick) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float corr = 0.f;
    const long long st = ticks[i];
    if (!(active && active[i]) && (float)st > 4.f * lim[i]) {       // lim is finite here
      const double l4 = fmax((double)(4.f * lim[i]), 1.0);
      const long long s2 = 1ll << (int)floor(log2(l4));
      const long long old_end = begin[i] + st;
      const long long new_end = min((ti_end / s2 + 1) * s2, old_end);
      if (new_end < old_end) {
        const long long nl = new_end - begin[i];
        corr = (float)((double)(nl - st) * 0.5 * dt_min);
        ticks[i] = nl;
      }
    }
    kick[i] = corr;
  }
}
