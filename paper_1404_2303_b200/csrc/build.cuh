// build.cuh — neighbour-finding structure on the device (section 3.2-3.3).
//
//  a1  k_hrange / k_validate_x  : max/min h_build, domain checks
//  a2  k_keys                   : key = top-cell index | Morton octants to `depth` levels,
//                                 sorted by the radix sort (radix_sort.cuh)
//  a3  k_gather_build           : particles packed in cell order (float4 {x,y,z,h})
//  a4  k_level_split / k_make_children : recursive split, "more than some minimal number"
//                                 and "a reasonable fraction" with h < edge/2 (P:510-518,
//                                 constants P:1354-1356), one level per launch
//  a5  k_top_slots / k_child_slots : every cell's 26 same-level neighbours (periodic at the
//                                 top; children inherit them through their
//                                 parent, which is the self refinement into 8 child selfs +
//                                 28 sibling pairs of P:519-522 and the pair refinement of
//                                 P:523-532).
//      k_tau / k_level_counts / k_list_masks : the interaction level of each particle.
//                                 tau_i = min(leaf level, deepest level with edge >= h_i).
//                                 The pair {i,j} is enumerated exactly once, at level
//                                 min(tau_i, tau_j), between the cells of i and j at that level
//                                 (equal or adjacent since r < max(h) <= edge). This is the
//                                 paper's refinement rule ("refine iff all h < edge/2")
//                                 applied per particle instead of per cell pair: the large-h
//                                 particles stay at the coarse level as a residue while the
//                                 rest of the pair is refined. Per cell and level
//                                 two source lists: A = {tau >= l} (targets with tau == l
//                                 sweep them) and R = {tau == l} (deeper targets sweep them).
//  a6  k_sort_warp / k_sort_block / big radix path : the A and R lists of each cell sorted
//                                 along the 13 canonical axes where a neighbour needs them
//                                 (P:687-698), plus an unsorted copy for the cell's own sweep
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
  int* nA;          // #{i in cell : tau_i >= level}   (list A)
  int* nR;          // #{i in cell : tau_i == level}   (list R)
  int* amask;       // 14-bit: directions 0..12 (+ bit 13 unsorted) of list A that are needed
  int* rmask;       // 14-bit, list R
  int64_t* offA;    // offsets of the node's A / R blocks in the list array (see k_list_masks)
  int64_t* offR;
  float* hmaxA;     // max final h over list A / R (force window)
  float* hmaxR;
};
#define LIST_SELF 13  // "direction" of the unsorted copy used for the cell's own sweep

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

// slots of the nodes of level l >= 1 from their parent's slots (gather form: no atomics).
// Every existing same-level neighbour is recorded; which pairs a level enumerates is
// decided per particle by tau (k_tau), not per cell pair.
__global__ void k_child_slots(int a, int b, NodeArrays N) {
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
        if (Y >= 0) y = N.child[8 * (int64_t)Y + bo];              // pair refinement
      }
    }
    N.slot[27 * (int64_t)c + k] = y;
  }
}

// tau_i = min(leaf level, deepest level l with min edge E_l >= h_build,i): at that level
// every partner j with r < max(h_i, h_j) and tau_j >= tau_i lies in the 27 cells around i.
__global__ void k_tau(int nnodes, NodeArrays N, LevelGeom g, const float* __restrict__ hb,
                      uint8_t* __restrict__ tau) {
  const int lane = threadIdx.x & 31;
  const int node = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= nnodes || N.split[node]) return;
  const int first = N.first[node], cnt = N.count[node], L = N.ijk[node].w;
  for (int s = first + lane; s < first + cnt; s += 32) {
    const float h = hb[s] * 1.000001f;
    int t = L;
    while (t > 0 && 2.f * g.half_min[t] < h) --t;
    tau[s] = (uint8_t)t;
  }
}

__global__ void k_level_counts(int nnodes, NodeArrays N, const uint8_t* __restrict__ tau) {
  const int lane = threadIdx.x & 31;
  const int node = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= nnodes) return;
  const int first = N.first[node], cnt = N.count[node], l = N.ijk[node].w;
  int na = 0, nr = 0;
  for (int s = first + lane; s < first + cnt; s += 32) {
    const int t = tau[s];
    na += t >= l;
    nr += t == l;
  }
  na = warp_sum_i(na);
  nr = warp_sum_i(nr);
  if (lane == 0) {
    N.nA[node] = na;
    N.nR[node] = nr;
  }
}

// which lists a cell must provide as a source: its neighbour X (or itself, bit 13) sweeps
// list A of this cell if X has targets with tau == l, list R if X has targets with tau > l.
// A direction is stored presorted only if the list is longer than sort_min_len
// and at least SORT_DEMAND_MIN targets sweep it; otherwise the sweeping warps read the whole
// list with the box filter alone: a warp stages 32 sources at a time, so a sorted window
// cannot save anything on a list of a few chunks, and sorting a list that one or two warps
// visit costs more than it saves. An unsorted sweep reads a compacted copy (bit 13), or,
// when every particle of the cell is a member (bit 14), the cell's own contiguous range.
#define SORT_DEMAND_MIN 64
#define LIST_RANGE 14
__global__ void k_list_masks(int nnodes, NodeArrays N, int sort_min_len, int64_t* __restrict__ nsort /*[2*nnodes]*/) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= nnodes) return;
  const int na = N.nA[y], nr = N.nR[y], cnt = N.count[y];
  (void)cnt;
  int demA[14], demR[14];
#pragma unroll
  for (int d = 0; d < 14; ++d) demA[d] = demR[d] = 0;
  for (int k = 0; k < 27; ++k) {
    const int x = (k == 13) ? y : N.slot[27 * (int64_t)y + k];
    if (x < 0) continue;
    const int d = (k == 13) ? LIST_SELF : slot_dir(k);
    demA[d] += N.nR[x];
    demR[d] += N.nA[x] - N.nR[x];
  }
  const int uR = (nr == cnt) ? (1 << LIST_RANGE) : (1 << LIST_SELF);
  int am = 0, rm = 0;
#pragma unroll
  for (int d = 0; d < 14; ++d) {
    // list A (tau >= l) is never stored: it is swept as the cell's own range, culled down its
    // sub-cells to the targets' reach and filtered by tau (cull_range) -- a 3D filter that
    // beats a 1D projection window, so sorting it would not pay.
    // With sort_min_len == 0 it is presorted along every swept direction (paper-literal).
    if (na > 0 && demA[d] > 0) {
      const bool srt = d != LIST_SELF && sort_min_len == 0;
      am |= srt ? (1 << d) : (1 << LIST_RANGE);
    }
    if (nr > 0 && demR[d] > 0) {
      const bool srt = d != LIST_SELF && (sort_min_len == 0 || (demR[d] >= SORT_DEMAND_MIN && nr > sort_min_len));
      rm |= srt ? (1 << d) : uR;
    }
  }
  N.amask[y] = am;
  N.rmask[y] = rm;
  nsort[2 * (int64_t)y] = (int64_t)__popc(am & 0x3fff) * na;
  nsort[2 * (int64_t)y + 1] = (int64_t)__popc(rm & 0x3fff) * nr;
}

__global__ void k_split_offsets(int nnodes, const int64_t* __restrict__ scan2, NodeArrays N) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= nnodes) return;
  N.offA[y] = scan2[2 * (int64_t)y];
  N.offR[y] = scan2[2 * (int64_t)y + 1];
}

// ---------------------------------------------------------------- a6 ---------
__device__ __forceinline__ float proj(float rx, float ry, float rz, float3 d) {
  return fmaf(rx, d.x, fmaf(ry, d.y, rz * d.z));
}

struct SortEntry {  // 8 bytes: projection key and cell-order particle index
  float key;
  int idx;
};

struct ListSeg {     // one (cell, kind) list family: members, directions, destination
  int cnt, mask;
  int64_t off;
};
__device__ __forceinline__ ListSeg list_seg(const NodeArrays& N, int node, int kind) {
  ListSeg L;
  L.cnt = kind ? N.nR[node] : N.nA[node];
  L.mask = kind ? N.rmask[node] : N.amask[node];
  L.off = kind ? N.offR[node] : N.offA[node];
  return L;
}
__device__ __forceinline__ bool list_member(int t, int l, int kind) { return kind ? (t == l) : (t >= l); }

// warp per (node, kind) with node count <= 32: one particle per lane, warp bitonic sort
__global__ void k_sort_warp(int nnodes, const float4* __restrict__ xh, const uint8_t* __restrict__ tau,
                            NodeArrays N, LevelGeom g, SortEntry* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int node = (int)(wid >> 1), kind = (int)(wid & 1);
  if (node >= nnodes) return;
  const ListSeg L = list_seg(N, node, kind);
  const int cnt_node = N.count[node];
  if ((L.mask & 0x3fff) == 0 || L.cnt == 0 || cnt_node > 32) return;
  const int first = N.first[node];
  const int4 c = N.ijk[node];
  float rx = 0.f, ry = 0.f, rz = 0.f;
  bool mem = false;
  if (lane < cnt_node) {
    float4 p = xh[first + lane];
    rx = p.x - node_corner(c.x, c.w, 0, g);
    ry = p.y - node_corner(c.y, c.w, 1, g);
    rz = p.z - node_corner(c.z, c.w, 2, g);
    mem = list_member(tau[first + lane], c.w, kind);
  }
  int r = 0;
  for (int d = 0; d < 14; ++d) {
    if (!((L.mask >> d) & 1)) continue;
    float key = (d == LIST_SELF) ? 0.f : proj(rx, ry, rz, dir_unit(d));
    uint64_t v = mem ? (((uint64_t)float_ord(key) << 32) | (uint32_t)lane) : ~0ull;
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
    int li = (lane < L.cnt) ? (int)(uint32_t)v : 0;
    float kk = __shfl_sync(FULL_MASK, key, li);
    if (lane < L.cnt) out[L.off + (int64_t)r * L.cnt + lane] = SortEntry{kk, first + li};
    ++r;
  }
}

// deterministic block compaction of the members of (node, kind) into smem (cell order)
__device__ __forceinline__ int block_compact_members(int first, int cnt_node, int l, int kind,
                                                     const uint8_t* __restrict__ tau, int* mem, int cap,
                                                     int* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int total = 0;
  for (int base = 0; base < cnt_node; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool m = i < cnt_node && list_member(tau[first + i], l, kind);
    const unsigned bal = __ballot_sync(FULL_MASK, m);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int before = 0;
    for (int ww = 0; ww < w; ++ww) before += wsum[ww];
    int tot = 0;
    for (int ww = 0; ww < nw; ++ww) tot += wsum[ww];
    const int pos = total + before + __popc(bal & lanemask_lt());
    if (m && pos < cap) mem[pos] = i;
    total += tot;
    __syncthreads();
  }
  return total;
}

#define SORT_BLOCK_MAX 4096
// CTA per (node, kind) with 32 < node count and members <= SORT_BLOCK_MAX: shared-memory
// bitonic sort per direction of (key, member index) composites
__global__ void __launch_bounds__(512) k_sort_block(int nnodes, const float4* __restrict__ xh,
                                                     const uint8_t* __restrict__ tau, NodeArrays N, LevelGeom g,
                                                     SortEntry* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sb_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(sb_raw);
  float* skey = reinterpret_cast<float*>(sk + SORT_BLOCK_MAX);
  int* mem = reinterpret_cast<int*>(skey + SORT_BLOCK_MAX);
  __shared__ int wsum[32];
  const int node = blockIdx.x >> 1, kind = blockIdx.x & 1;
  if (node >= nnodes) return;
  const ListSeg L = list_seg(N, node, kind);
  const int cnt_node = N.count[node];
  if ((L.mask & 0x3fff) == 0 || L.cnt == 0 || cnt_node <= 32 || L.cnt > SORT_BLOCK_MAX) return;
  const int first = N.first[node];
  const int4 c = N.ijk[node];
  block_compact_members(first, cnt_node, c.w, kind, tau, mem, SORT_BLOCK_MAX, wsum);
  const int cnt = L.cnt;
  const float cx = node_corner(c.x, c.w, 0, g), cy = node_corner(c.y, c.w, 1, g),
              cz = node_corner(c.z, c.w, 2, g);
  int P = 64;
  while (P < cnt) P <<= 1;
  int r = 0;
  for (int d = 0; d < 14; ++d) {
    if (!((L.mask >> d) & 1)) continue;
    if (d == LIST_SELF) {
      for (int i = threadIdx.x; i < cnt; i += blockDim.x)
        out[L.off + (int64_t)r * cnt + i] = SortEntry{0.f, first + mem[i]};
      ++r;
      continue;
    }
    float3 dv = dir_unit(d);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < cnt) {
        float4 p = xh[first + mem[i]];
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
      out[L.off + (int64_t)r * cnt + i] = SortEntry{skey[li], first + mem[li]};
    }
    __syncthreads();
    ++r;
  }
}

// big lists (members > SORT_BLOCK_MAX): composite keys (segment, key) for the radix sort.
// Segment ids grow with the destination offset, so the sorted order is the layout order.
__global__ void __launch_bounds__(512) k_big_keys(int nbig, const int* __restrict__ bigseg,
                                                  const int64_t* __restrict__ bigoff, const float4* __restrict__ xh,
                                                  const uint8_t* __restrict__ tau, NodeArrays N, LevelGeom g,
                                                  uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  __shared__ int wsum[32];
  const int bi = blockIdx.x;
  if (bi >= nbig) return;
  const int node = bigseg[bi] >> 1, kind = bigseg[bi] & 1;
  const ListSeg L = list_seg(N, node, kind);
  const int first = N.first[node], cnt_node = N.count[node];
  const int4 c = N.ijk[node];
  const float cx = node_corner(c.x, c.w, 0, g), cy = node_corner(c.y, c.w, 1, g),
              cz = node_corner(c.z, c.w, 2, g);
  const int64_t base = bigoff[bi];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int total = 0;
  for (int b0 = 0; b0 < cnt_node; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    const bool m = i < cnt_node && list_member(tau[first + i], c.w, kind);
    const unsigned bal = __ballot_sync(FULL_MASK, m);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int ww = 0; ww < nw; ++ww) {
      if (ww < w) before += wsum[ww];
      tot += wsum[ww];
    }
    if (m) {
      const int pos = total + before + __popc(bal & lanemask_lt());
      const float4 p = xh[first + i];
      int r = 0;
      for (int d = 0; d < 14; ++d) {
        if (!((L.mask >> d) & 1)) continue;
        const float key = (d == LIST_SELF) ? 0.f : proj(p.x - cx, p.y - cy, p.z - cz, dir_unit(d));
        const uint64_t seg = (uint64_t)bi * 14 + r;
        keys[base + (int64_t)r * L.cnt + pos] = (seg << 32) | float_ord(key);
        vals[base + (int64_t)r * L.cnt + pos] = (uint32_t)(first + i);
        ++r;
      }
    }
    total += tot;
    __syncthreads();
  }
}

__device__ __forceinline__ float ord_float(uint32_t u) {
  uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(b);
}

__global__ void k_big_write(int nbig, const int* __restrict__ bigseg, const int64_t* __restrict__ bigoff,
                            NodeArrays N, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                            SortEntry* __restrict__ out) {
  int bi = blockIdx.x;
  if (bi >= nbig) return;
  const ListSeg L = list_seg(N, bigseg[bi] >> 1, bigseg[bi] & 1);
  int64_t n_ent = (int64_t)__popc(L.mask & 0x3fff) * L.cnt;
  int64_t src = bigoff[bi];
  for (int64_t i = threadIdx.x; i < n_ent; i += blockDim.x)
    out[L.off + i] = SortEntry{ord_float((uint32_t)keys[src + i]), (int)vals[src + i]};
}

__global__ void k_mark_big(int nnodes, NodeArrays N, int* __restrict__ flag, int64_t* __restrict__ sz) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 2 * nnodes) return;
  const ListSeg L = list_seg(N, x >> 1, x & 1);
  bool big = (L.mask & 0x3fff) != 0 && L.cnt > SORT_BLOCK_MAX;
  flag[x] = big ? 1 : 0;
  sz[x] = big ? (int64_t)__popc(L.mask & 0x3fff) * L.cnt : 0;
}

__global__ void k_compact_big(int nseg, const int* __restrict__ flag, const int* __restrict__ idx,
                              const int64_t* __restrict__ szscan, int* __restrict__ bigseg,
                              int64_t* __restrict__ bigoff) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nseg || !flag[x]) return;
  bigseg[idx[x]] = x;
  bigoff[idx[x]] = szscan[x];
}

// Per target cell X and kind (0: A-lists for targets with tau == level, 1: R-lists for
// deeper targets): the non-empty source lists of the 27 cells around X, as descriptors
// with the list offset for the sweep direction, the periodic shift and Y's corner.
struct SegDesc {   // 32 bytes
  long long off;   // first entry of the list in the sweep direction
  int cnt;         // entries
  int meta;        // bits 0-4 k (slot), 5 flip, 6 self (k == 13), 7 swept whole (no window),
                   // 8-13 shift codes (2 bits/axis: 1 = +1, 2 = -1), 14 list = cell range,
                   // 15 range holds non-members (keep tau >= level only), 16-19 dir
  float cx, cy, cz;  // Y's corner + source shift (frame of the keys)
  int Y;
};

__device__ __forceinline__ bool seg_needed(const NodeArrays& N, int X, int kind) {
  return kind ? (N.nA[X] - N.nR[X]) > 0 : N.nR[X] > 0;
}

__global__ void k_seg_count(int nnodes, NodeArrays N, int* __restrict__ cnt2) {
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= nnodes) return;
  for (int kind = 0; kind < 2; ++kind) {
    int c = 0;
    if (seg_needed(N, X, kind)) {
      for (int k = 0; k < 27; ++k) {
        const int Y = (k == 13) ? X : N.slot[27 * (int64_t)X + k];
        if (Y >= 0 && (kind ? N.nR[Y] : N.nA[Y]) > 0) ++c;
      }
    }
    cnt2[2 * X + kind] = c;
  }
}

__global__ void k_seg_fill(int nnodes, NodeArrays N, LevelGeom g, const int* __restrict__ off2,
                           SegDesc* __restrict__ out) {
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= nnodes) return;
  const int4 cX = N.ijk[X];
  const int l = cX.w;
  for (int kind = 0; kind < 2; ++kind) {
    if (!seg_needed(N, X, kind)) continue;
    int o = off2[2 * X + kind];
    for (int k = 0; k < 27; ++k) {
      const int Y = (k == 13) ? X : N.slot[27 * (int64_t)X + k];
      if (Y < 0) continue;
      const ListSeg L = list_seg(N, Y, kind);
      if (L.cnt == 0) continue;
      int d = (k == 13) ? LIST_SELF : slot_dir(k);
      const bool unsorted = (d == LIST_SELF) || !((L.mask >> d) & 1);   // swept whole, no window
      const bool range = unsorted && ((L.mask >> LIST_RANGE) & 1);       // = the cell's own range
      const bool tfilter = range && kind == 0 && N.nA[Y] != N.count[Y];  // range holds non-members
      if (unsorted) d = LIST_SELF;
      SegDesc sd;
      sd.off = range ? (long long)N.first[Y] : L.off + (long long)__popc(L.mask & ((1 << d) - 1)) * L.cnt;
      sd.cnt = range ? N.count[Y] : L.cnt;
      sd.Y = Y;
      int meta = k | (slot_flip(k) ? 32 : 0) | (k == 13 ? 64 : 0) | (unsorted ? 128 : 0) | (range ? (1 << 14) : 0) |
                 (tfilter ? (1 << 15) : 0) | (d << 16);
      float so[3] = {0.f, 0.f, 0.f};
      if (k != 13) {
        const int4 cY = N.ijk[Y];
        const int dd[3] = {cX.x + off_x(k) - cY.x, cX.y + off_y(k) - cY.y, cX.z + off_z(k) - cY.z};
        for (int a = 0; a < 3; ++a) {
          const int sa = dd[a] > 1 ? 1 : (dd[a] < -1 ? -1 : 0);
          meta |= (sa > 0 ? 1 : (sa < 0 ? 2 : 0)) << (8 + 2 * a);
          so[a] = sa < 0 ? -g.L[a] : 0.f;
        }
        sd.cx = node_corner(cY.x, l, 0, g) + so[0];
        sd.cy = node_corner(cY.y, l, 1, g) + so[1];
        sd.cz = node_corner(cY.z, l, 2, g) + so[2];
      } else {
        sd.cx = sd.cy = sd.cz = 0.f;
      }
      sd.meta = meta;
      out[o++] = sd;
    }
  }
}

// ---------------------------------------------------------------- tasks ------
// Work unit of the interaction kernels: a leaf cell's particles in chunks of 32 (cell order).
__global__ void k_leaf_chunks(int nnodes, NodeArrays N, int* __restrict__ nchunk) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  nchunk[x] = N.split[x] ? 0 : (N.count[x] + 31) >> 5;
}

__global__ void k_write_tasks(int nnodes, NodeArrays N, const int* __restrict__ nchunk, const int* __restrict__ scan,
                              int4* __restrict__ tasks) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nnodes) return;
  const int c = nchunk[x], b = scan[x], first = N.first[x], cnt = N.count[x];
  for (int i = 0; i < c; ++i) tasks[b + i] = make_int4(x, first + 32 * i, min(32, cnt - 32 * i), 0);
}

// per node max of the final h over lists A and R (force window)
__global__ void k_node_hmax(int nnodes, NodeArrays N, const float4* __restrict__ xh, const uint8_t* __restrict__ tau) {
  const int lane = threadIdx.x & 31;
  const int node = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (node >= nnodes) return;
  const int first = N.first[node], cnt = N.count[node], l = N.ijk[node].w;
  float ha = 0.f, hr = 0.f;
  for (int s = first + lane; s < first + cnt; s += 32) {
    const int t = tau[s];
    const float h = xh[s].w;
    if (t >= l) ha = fmaxf(ha, h);
    if (t == l) hr = fmaxf(hr, h);
  }
  ha = warp_max_f(ha);
  hr = warp_max_f(hr);
  if (lane == 0) {
    N.hmaxA[node] = ha;
    N.hmaxR[node] = hr;
  }
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
