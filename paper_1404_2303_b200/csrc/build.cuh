// build.cuh — neighbour-finding structure on the device (section 3.2-3.3).
//
//  a1  k_hrange / k_validate_x  : max/min h_build, domain checks
//  a2  k_keys                   : key = top-cell index | Morton octants to `depth` levels,
//                                 sorted by the radix sort (radix_sort.cuh)
//  a3  k_gather_build           : particles packed in cell order (float4 {x,y,z,h})
//  a4  k_level_split / k_make_children : recursive split, "more than some minimal number"
//                                 and "a reasonable fraction" with h < edge/2 (P:510-518,
//                                 constants P:1354-1356), one level per launch
//  a5  k_top_slots / k_child_slots / k_kept : interaction slots. Top cells pair with their
//                                 26 periodic neighbours; a split cell's self
//                                 becomes 8 child selfs + 28 sibling pairs;
//                                 a pair is refined iff both cells are split and all h in
//                                 both are < edge/2, else kept whole.
//  a6  k_sort_warp / k_sort_block / big-node radix path : per (cell, direction) lists
//                                 sorted along the 13 canonical axes
#pragma once
#include "common.cuh"

struct NodeArrays {
  int* first;       // first particle (cell order)
  int* count;
  int4* ijk;        // integer cell coordinates at its level, .w = level
  int* parent;
  int* child;       // [8*node + octant], -1 if empty / leaf
  float* hmaxb;     // max h_build in the cell
  int* split;       // 1 if split into children
  int* slot;        // [27*node + k] neighbour cell at offset k (same level), -1 if none
  int* kept;        // 27-bit mask of kept pair slots
  int* dirmask;     // 13-bit mask of sorted directions needed (as a source)
  int64_t* sortoff; // offset of the node's sorted block in the list array
  float* hmaxf;     // max final h in the cell (force window)
};

struct LevelGeom {           // per-level edges (fp32), up to SPH_MAX_DEPTH+1 levels
  float E[SPH_MAX_DEPTH + 2][3];
  float half_min[SPH_MAX_DEPTH + 2];   // min_k E_l,k / 2
  int n[SPH_MAX_DEPTH + 2][3];         // cells per axis at level l (ntop << l)
  float L[3];
  int depth;
};

__host__ __device__ __forceinline__ float node_corner(int i, int l, int axis, const LevelGeom& g) {
  return (float)((double)i * (double)g.E[l][axis]);
}

// ---------------------------------------------------------------- a1 ---------
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

__global__ void k_hrange(const float* __restrict__ h, int64_t n, unsigned long long* ctr) {
  unsigned mx = 0u, mn = 0x7f800000u;
  int err = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = h[i];
    if (!isfinite(v) || v < 0.f) err |= ERRBIT_H;
    else if (v > 0.f) {
      unsigned b = __float_as_uint(v);
      mx = max(mx, b);
      mn = min(mn, b);
    }
  }
  mx = __reduce_max_sync(FULL_MASK, mx);
  mn = __reduce_min_sync(FULL_MASK, mn);
  err = __reduce_or_sync(FULL_MASK, err);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&ctr[C_HMAXBITS], (unsigned long long)mx);
    atomicMin(&ctr[C_HMINBITS], (unsigned long long)mn);
    if (err) atomicOr(&ctr[C_ERR], (unsigned long long)err);
  }
}

// ---------------------------------------------------------------- a2 ---------
__global__ void k_keys(const float* __restrict__ x, int64_t n, int nx, int ny, int nz, int depth,
                       double sx, double sy, double sz, uint64_t* __restrict__ keys,
                       uint32_t* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fx = ((int64_t)nx << depth) - 1, fy = ((int64_t)ny << depth) - 1,
                  fz = ((int64_t)nz << depth) - 1;
    int64_t cx = (int64_t)floor((double)x[3 * i] * sx);
    int64_t cy = (int64_t)floor((double)x[3 * i + 1] * sy);
    int64_t cz = (int64_t)floor((double)x[3 * i + 2] * sz);
    cx = min(max(cx, (int64_t)0), fx);
    cy = min(max(cy, (int64_t)0), fy);
    cz = min(max(cz, (int64_t)0), fz);
    uint64_t t = (uint64_t)((cx >> depth) + (int64_t)nx * ((cy >> depth) + (int64_t)ny * (cz >> depth)));
    uint64_t m = 0;
    for (int b = depth - 1; b >= 0; --b) {
      uint64_t oct = (((cx >> b) & 1) << 2) | (((cy >> b) & 1) << 1) | ((cz >> b) & 1);
      m = (m << 3) | oct;
    }
    keys[i] = (t << (3 * depth)) | m;
    vals[i] = (uint32_t)i;
  }
}

// ---------------------------------------------------------------- a3 ---------
__global__ void k_gather_build(const uint32_t* __restrict__ perm, int64_t n, const float* __restrict__ x,
                               const float* __restrict__ hcur, const float* __restrict__ hb_o,
                               const float* __restrict__ lo_o, const float* __restrict__ hi_o,
                               float4* __restrict__ xh, float* __restrict__ hb, float* __restrict__ lo,
                               float* __restrict__ hi) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    uint32_t p = perm[s];
    xh[s] = make_float4(x[3 * (int64_t)p], x[3 * (int64_t)p + 1], x[3 * (int64_t)p + 2], hcur[p]);
    hb[s] = hb_o[p];
    if (lo) lo[s] = lo_o[p];
    if (hi) hi[s] = hi_o[p];
  }
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

__global__ void k_top_counts(int n0, int64_t n, NodeArrays N) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n0) N.count[i] = (i + 1 < n0 ? N.first[i + 1] : (int)n) - N.first[i];
}

// ---------------------------------------------------------------- a4 ---------
// warp per node of one level: h_build max, fraction with h < edge/2, split decision
// (P:510-518), child boundaries by binary search on the octant bits.
__global__ void k_level_split(int a, int b, int level, int depth, const float* __restrict__ hb,
                              const uint64_t* __restrict__ keys, float half_edge, int split_count,
                              float split_frac, int count_only, NodeArrays N, int* __restrict__ nch,
                              int* __restrict__ chstart) {
  const int lane = threadIdx.x & 31;
  const int node = a + (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= b) return;
  const int first = N.first[node], cnt = N.count[node];
  float hm = 0.f;
  int nsmall = 0;
  for (int s = first + lane; s < first + cnt; s += 32) {
    float h = hb[s];
    hm = fmaxf(hm, h);
    nsmall += (h < half_edge) ? 1 : 0;
  }
  hm = warp_max_f(hm);
  nsmall = warp_sum_i(nsmall);
  int sp = (level < depth) && (cnt > split_count) &&
           (count_only || (double)nsmall > (double)split_frac * (double)cnt);
  if (lane == 0) {
    N.hmaxb[node] = hm;
    N.split[node] = sp;
  }
  if (!sp) {
    if (lane == 0) nch[node - a] = 0;
    return;
  }
  const int shift = 3 * (depth - level - 1);
  int start = first + cnt;
  if (lane < 8) {
    int lo = first, hi = first + cnt;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      int oct = (int)((keys[mid] >> shift) & 7ull);
      if (oct < lane) lo = mid + 1;
      else hi = mid;
    }
    start = lo;
  }
  int nxt = __shfl_down_sync(FULL_MASK, start, 1);
  int ne = (lane < 8 && nxt - start > 0) ? 1 : 0;
  unsigned bal = __ballot_sync(FULL_MASK, ne);
  if (lane < 8) chstart[8 * (int64_t)node + lane] = start;
  if (lane == 0) nch[node - a] = __popc(bal);
}

__global__ void k_make_children(int a, int b, int64_t n_first_next, const int* __restrict__ nch,
                                 const int* __restrict__ chscan, NodeArrays N) {
  int p = a + blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= b) return;
  int* ch = N.child + 8 * (int64_t)p;
  if (nch[p - a] == 0) {
#pragma unroll
    for (int o = 0; o < 8; ++o) ch[o] = -1;
    return;
  }
  int st[9];
#pragma unroll
  for (int o = 0; o < 8; ++o) st[o] = ch[o];
  st[8] = N.first[p] + N.count[p];
  int4 pijk = N.ijk[p];
  int k = 0;
  int base = (int)(n_first_next + chscan[p - a]);
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    int c = st[o + 1] - st[o];
    if (c > 0) {
      int cn = base + k++;
      N.first[cn] = st[o];
      N.count[cn] = c;
      N.ijk[cn] = make_int4(2 * pijk.x + ((o >> 2) & 1), 2 * pijk.y + ((o >> 1) & 1),
                            2 * pijk.z + (o & 1), pijk.w + 1);
      N.parent[cn] = p;
      ch[o] = cn;
    } else {
      ch[o] = -1;
    }
  }
}

// ---------------------------------------------------------------- a5 ---------
__global__ void k_top_slots(int n0, int nx, int ny, int nz, const int* __restrict__ topmap, NodeArrays N) {
  int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= n0) return;
  int4 c = N.ijk[node];
  for (int k = 0; k < 27; ++k) {
    int y = -1;
    if (k != 13) {
      int ix = (c.x + off_x(k) + nx) % nx, iy = (c.y + off_y(k) + ny) % ny, iz = (c.z + off_z(k) + nz) % nz;
      y = topmap[ix + (int64_t)nx * (iy + (int64_t)ny * iz)];
    }
    N.slot[27 * (int64_t)node + k] = y;
  }
}

__device__ __forceinline__ bool refine_pair(const NodeArrays& N, int x, int y, float half_edge) {
  return N.split[x] && N.split[y] && N.hmaxb[x] < half_edge && N.hmaxb[y] < half_edge;
}

// slots of the nodes of level l >= 1 from their parent's slots (gather form: no atomics)
__global__ void k_child_slots(int a, int b, float parent_half_edge, NodeArrays N) {
  int c = a + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= b) return;
  int X = N.parent[c];
  int4 ijk = N.ijk[c];
  int ax = ijk.x & 1, ay = ijk.y & 1, az = ijk.z & 1;
  for (int k = 0; k < 27; ++k) {
    int y = -1;
    if (k != 13) {
      int tx = ax + off_x(k), ty = ay + off_y(k), tz = az + off_z(k);
      int Px = tx < 0 ? -1 : (tx >> 1), Py = ty < 0 ? -1 : (ty >> 1), Pz = tz < 0 ? -1 : (tz >> 1);
      int bo = ((tx - 2 * Px) << 2) | ((ty - 2 * Py) << 1) | (tz - 2 * Pz);
      if (Px == 0 && Py == 0 && Pz == 0) {
        y = N.child[8 * (int64_t)X + bo];                          // sibling (self refinement)
      } else {
        int kp = (Px + 1) * 9 + (Py + 1) * 3 + (Pz + 1);
        int Y = N.slot[27 * (int64_t)X + kp];
        if (Y >= 0 && refine_pair(N, X, Y, parent_half_edge)) y = N.child[8 * (int64_t)Y + bo];
      }
    }
    N.slot[27 * (int64_t)c + k] = y;
  }
}

// kept pair slots and the sorted directions each cell needs as a source
__global__ void k_kept(int a, int b, float half_edge, NodeArrays N, int64_t* __restrict__ nsort) {
  int x = a + blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= b) return;
  int kept = 0, dm = 0;
  for (int k = 0; k < 27; ++k) {
    int y = N.slot[27 * (int64_t)x + k];
    if (y >= 0 && !refine_pair(N, x, y, half_edge)) {
      kept |= 1 << k;
      dm |= 1 << slot_dir(k);
    }
  }
  N.kept[x] = kept;
  N.dirmask[x] = dm;
  nsort[x] = (int64_t)__popc(dm) * N.count[x];
}

// ---------------------------------------------------------------- a6 ---------
__device__ __forceinline__ float proj(float rx, float ry, float rz, float3 d) {
  return fmaf(rx, d.x, fmaf(ry, d.y, rz * d.z));
}

struct SortEntry {  // 8 bytes: projection key and cell-order particle index
  float key;
  int idx;
};

// warp per node with count <= 32: one particle per lane, warp bitonic sort per direction
__global__ void k_sort_warp(int nnodes, const float4* __restrict__ xh, NodeArrays N, LevelGeom g,
                            SortEntry* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int node = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= nnodes) return;
  const int cnt = N.count[node];
  const int dm = N.dirmask[node];
  if (dm == 0 || cnt > 32) return;
  const int first = N.first[node];
  const int4 c = N.ijk[node];
  float rx = 0.f, ry = 0.f, rz = 0.f;
  if (lane < cnt) {
    float4 p = xh[first + lane];
    rx = p.x - node_corner(c.x, c.w, 0, g);
    ry = p.y - node_corner(c.y, c.w, 1, g);
    rz = p.z - node_corner(c.z, c.w, 2, g);
  }
  int64_t base = N.sortoff[node];
  int r = 0;
  for (int d = 0; d < 13; ++d) {
    if (!((dm >> d) & 1)) continue;
    float key = proj(rx, ry, rz, dir_unit(d));
    uint64_t v = (lane < cnt) ? (((uint64_t)float_ord(key) << 32) | (uint32_t)lane) : ~0ull;
    // bitonic sort of 32 values across the warp (ascending)
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
    int li = (lane < cnt) ? (int)(uint32_t)v : 0;
    float kk = __shfl_sync(FULL_MASK, key, li);
    if (lane < cnt) out[base + (int64_t)r * cnt + lane] = SortEntry{kk, first + li};
    ++r;
  }
}

#define SORT_BLOCK_MAX 4096
// CTA per node with 32 < count <= SORT_BLOCK_MAX: shared-memory bitonic sort per direction
__global__ void __launch_bounds__(512) k_sort_block(int nnodes, const float4* __restrict__ xh, NodeArrays N,
                                                     LevelGeom g, SortEntry* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sb_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(sb_raw);
  float* skey = reinterpret_cast<float*>(sk + SORT_BLOCK_MAX);
  const int node = blockIdx.x;
  if (node >= nnodes) return;
  const int cnt = N.count[node];
  const int dm = N.dirmask[node];
  if (dm == 0 || cnt <= 32 || cnt > SORT_BLOCK_MAX) return;
  const int first = N.first[node];
  const int4 c = N.ijk[node];
  const float cx = node_corner(c.x, c.w, 0, g), cy = node_corner(c.y, c.w, 1, g),
              cz = node_corner(c.z, c.w, 2, g);
  int P = 64;
  while (P < cnt) P <<= 1;
  int64_t base = N.sortoff[node];
  int r = 0;
  for (int d = 0; d < 13; ++d) {
    if (!((dm >> d) & 1)) continue;
    float3 dv = dir_unit(d);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < cnt) {
        float4 p = xh[first + i];
        float key = proj(p.x - cx, p.y - cy, p.z - cz, dv);
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
          int lo = 2 * i - (i & (stride - 1));
          int hi = lo + stride;
          bool up = ((lo & size) == 0);
          uint64_t A = sk[lo], B = sk[hi];
          if ((A > B) == up) {
            sk[lo] = B;
            sk[hi] = A;
          }
        }
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      int li = (int)(uint32_t)sk[i];
      out[base + (int64_t)r * cnt + i] = SortEntry{skey[li], first + li};
    }
    __syncthreads();
    ++r;
  }
}

// big nodes (count > SORT_BLOCK_MAX): composite keys (segment, key) sorted by the radix sort
__global__ void k_big_keys(int nbig, const int* __restrict__ bignodes, const int64_t* __restrict__ bigoff,
                           const float4* __restrict__ xh, NodeArrays N, LevelGeom g,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  int bi = blockIdx.x;
  if (bi >= nbig) return;
  int node = bignodes[bi];
  int cnt = N.count[node], dm = N.dirmask[node], first = N.first[node];
  int4 c = N.ijk[node];
  const float cx = node_corner(c.x, c.w, 0, g), cy = node_corner(c.y, c.w, 1, g),
              cz = node_corner(c.z, c.w, 2, g);
  int64_t base = bigoff[bi];
  int r = 0;
  for (int d = 0; d < 13; ++d) {
    if (!((dm >> d) & 1)) continue;
    float3 dv = dir_unit(d);
    uint64_t seg = (uint64_t)bi * 13 + r;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      float4 p = xh[first + i];
      float key = proj(p.x - cx, p.y - cy, p.z - cz, dv);
      keys[base + (int64_t)r * cnt + i] = (seg << 32) | float_ord(key);
      vals[base + (int64_t)r * cnt + i] = (uint32_t)(first + i);
    }
    ++r;
  }
}

__device__ __forceinline__ float ord_float(uint32_t u) {
  uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(b);
}

__global__ void k_big_write(int nbig, const int* __restrict__ bignodes, const int64_t* __restrict__ bigoff,
                            NodeArrays N, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                            SortEntry* __restrict__ out) {
  int bi = blockIdx.x;
  if (bi >= nbig) return;
  int node = bignodes[bi];
  int64_t n_ent = (int64_t)__popc(N.dirmask[node]) * N.count[node];
  int64_t src = bigoff[bi], dst = N.sortoff[node];
  for (int64_t i = threadIdx.x; i < n_ent; i += blockDim.x)
    out[dst + i] = SortEntry{ord_float((uint32_t)keys[src + i]), (int)vals[src + i]};
}

__global__ void k_mark_big(int nnodes, NodeArrays N, int* __restrict__ flag, int64_t* __restrict__ sz) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  bool big = N.dirmask[x] != 0 && N.count[x] > SORT_BLOCK_MAX;
  flag[x] = big ? 1 : 0;
  sz[x] = big ? (int64_t)__popc(N.dirmask[x]) * N.count[x] : 0;
}

__global__ void k_compact_big(int nnodes, const int* __restrict__ flag, const int* __restrict__ idx,
                              const int64_t* __restrict__ szscan, int* __restrict__ bignodes,
                              int64_t* __restrict__ bigoff) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes || !flag[x]) return;
  bignodes[idx[x]] = x;
  bigoff[idx[x]] = szscan[x];
}

// ---------------------------------------------------------------- leaves -----
__global__ void k_leaf_chunks(int nnodes, NodeArrays N, int* __restrict__ nchunk) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  nchunk[x] = N.split[x] ? 0 : (N.count[x] + 31) >> 5;
}

__global__ void k_write_tasks(int nnodes, const int* __restrict__ nchunk, const int* __restrict__ scan,
                              int2* __restrict__ tasks) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  int c = nchunk[x], b = scan[x];
  for (int i = 0; i < c; ++i) tasks[b + i] = make_int2(x, i);
}

// per node max of the final h (force window)
__global__ void k_node_hmax(int nnodes, NodeArrays N, const float4* __restrict__ xh) {
  const int lane = threadIdx.x & 31;
  const int node = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= nnodes) return;
  int first = N.first[node], cnt = N.count[node];
  float hm = 0.f;
  for (int s = first + lane; s < first + cnt; s += 32) hm = fmaxf(hm, xh[s].w);
  hm = warp_max_f(hm);
  if (lane == 0) N.hmaxf[node] = hm;
}

// initial guess from cell occupancy: N = (4 pi/3) n h^3 for uniform density n (Eq. 3)
// -> h = cbrt(3 N_ngb / (4 pi n)); n from the leaf, or its parent if the leaf is sparse.
__global__ void k_guess_h(int nnodes, NodeArrays N, LevelGeom g, const uint32_t* __restrict__ perm,
                          float n_ngb, int min_count, float hcap, float* __restrict__ hguess_orig) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes || N.split[x]) return;
  int y = x;
  while (N.count[y] < min_count && N.parent[y] >= 0) y = N.parent[y];
  int l = N.ijk[y].w;
  double vol = (double)g.E[l][0] * g.E[l][1] * g.E[l][2];
  double dens = (double)N.count[y] / vol;
  float h = (float)cbrt(3.0 * n_ngb / (4.0 * 3.14159265358979323846 * dens));
  h = fminf(h, hcap);
  for (int s = N.first[x]; s < N.first[x] + N.count[x]; ++s) hguess_orig[perm[s]] = h;
}
