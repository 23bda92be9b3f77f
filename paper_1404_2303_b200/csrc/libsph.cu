// libsph.cu — host orchestration and the C ABI declared in include/sph.h.
// One translation unit (unity build) so every kernel is launched from the file that
// defines it; compiled for sm_100a only (see paper_1404_2303_b200/build.py).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <cstdlib>
#include <ctime>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"
#include "build.cuh"
#include "lists.cuh"
#include "interact.cuh"
#include "comm.cuh"
#include "integrate.cuh"
#include "ablation.cuh"

// =========================================================== memory =============
static void* dev_alloc(sph_ctx* c, size_t bytes) {
  if (c->ualloc) {
    void* p = c->ualloc(bytes, (void*)c->stream, c->uuser);
    SPH_REQUIRE(p != nullptr, SPH_E_OOM, "user allocator returned NULL");
    return p;
  }
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, bytes));
  return p;
}

static void dev_free(sph_ctx* c, void* p) {
  if (!p) return;
  if (c->ualloc) {
    c->urelease(p, (void*)c->stream, c->uuser);
  } else {
    cudaFree(p);
  }
}

// capacity-managed named buffer; keep=true preserves the old contents on growth
template <class T>
static T* B(sph_ctx* c, int id, size_t count, bool keep = false) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  DBuf& b = c->b[id];
  if (b.bytes < bytes) {
    size_t nb = std::max(bytes, b.bytes + b.bytes / 2);
    nb = (nb + 255) & ~size_t(255);
    void* np = dev_alloc(c, nb);
    if (keep && b.p) CUDA_TRY(cudaMemcpyAsync(np, b.p, b.bytes, cudaMemcpyDeviceToDevice, c->stream));
    if (b.p) {
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      dev_free(c, b.p);
    }
    b.p = np;
    b.bytes = nb;
  }
  return reinterpret_cast<T*>(b.p);
}
template <class T>
static T* Bget(sph_ctx* c, int id) {
  return reinterpret_cast<T*>(c->b[id].p);
}

#define LAUNCH(kern, grid, block, smem, ...)                                        \
  do {                                                                              \
    kern<<<(grid), (block), (smem), c->stream>>>(__VA_ARGS__);                      \
    c->launches++;                                                                  \
    CUDA_TRY(cudaGetLastError());                                                   \
  } while (0)

static int grid1d(sph_ctx* c, int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  g = std::min<int64_t>(g, (int64_t)c->num_sms * 16);
  return (int)std::max<int64_t>(g, 1);
}
static int gridfull(int64_t n, int block) { return (int)std::max<int64_t>((n + block - 1) / block, 1); }

static int64_t g_syncs = 0;
static void sync(sph_ctx* c) {
  ++g_syncs;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
}

static bool dbg_on() {
  const char* e = getenv("SPH_DEBUG");
  return e && e[0] && e[0] != '0';
}
#define DBG(...) do { if (dbg_on()) { fprintf(stderr, "[sph] " __VA_ARGS__); fflush(stderr); } } while (0)
// debug wall-clock of a region (device-synchronised), only when SPH_DEBUG is set
struct DbgTimer {
  sph_ctx* c;
  const char* what;
  double t0;
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  DbgTimer(sph_ctx* c_, const char* w) : c(c_), what(w), t0(0) {
    if (dbg_on()) {
      cudaStreamSynchronize(c->stream);
      t0 = now();
    }
  }
  ~DbgTimer() {
    if (dbg_on()) {
      cudaStreamSynchronize(c->stream);
      fprintf(stderr, "[sph]   %s: %.3f ms\n", what, now() - t0);
    }
  }
};

// =========================================================== phase timing =======
// events around the launches of a phase; resolved (summed into ms_phase) after a sync
struct PhaseTimer {
  sph_ctx* c;
  size_t k;
  cudaStream_t st;
  PhaseTimer(sph_ctx* c_, int phase, cudaStream_t s = nullptr) : c(c_), st(s ? s : c_->stream) {
    if (c->timed_used == c->timed.size()) {
      sph_ctx::Timed t;
      CUDA_TRY(cudaEventCreate(&t.a));
      CUDA_TRY(cudaEventCreate(&t.b));
      c->timed.push_back(t);
    }
    k = c->timed_used++;
    c->timed[k].phase = phase;
    CUDA_TRY(cudaEventRecord(c->timed[k].a, st));
  }
  ~PhaseTimer() { cudaEventRecord(c->timed[k].b, st); }
};
static void phase_resolve(sph_ctx* c) {
  for (size_t k = 0; k < c->timed_used; ++k) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->timed[k].a, c->timed[k].b);
    c->ms_phase[c->timed[k].phase] += ms;
  }
  c->timed_used = 0;
}
static void phase_reset(sph_ctx* c) {
  c->timed_used = 0;
  for (double& v : c->ms_phase) v = 0.0;
  c->nb_entries = 0;
  c->walk_launches = 0;
}

// =========================================================== counters ===========
static unsigned long long* ctr(sph_ctx* c) { return B<unsigned long long>(c, B_COUNTERS, C_NCOUNTERS); }
// a small device -> host read through the context's page-locked scratch (<= 64 words)
static void read_dev(sph_ctx* c, void* host, const void* dev, size_t bytes) {
  SPH_REQUIRE(bytes <= 64 * sizeof(unsigned long long), SPH_E_ARG, "read_dev: more than the pinned scratch");
  CUDA_TRY(cudaMemcpyAsync(c->hpin, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  memcpy(host, c->hpin, bytes);
}
// counters back to their initial values by a device-to-device copy (a host-to-device copy from
// pageable memory may wait for the stream)
static void ctr_reset(sph_ctx* c) {
  static const unsigned long long init[C_NCOUNTERS] = {0, 0, 0, 0, 0, 0, 0, 0x7f800000ull};   // C_HMINBITS = +inf
  static_assert(C_HMINBITS == 7, "counter layout");
  unsigned long long* d0 = B<unsigned long long>(c, B_CTRINIT, C_NCOUNTERS);
  if (!c->ctr_init_ready) {
    CUDA_TRY(cudaMemcpy(d0, init, sizeof(init), cudaMemcpyHostToDevice));
    c->ctr_init_ready = true;
  }
  CUDA_TRY(cudaMemcpyAsync(ctr(c), d0, sizeof(init), cudaMemcpyDeviceToDevice, c->stream));
}
static void ctr_read(sph_ctx* c, unsigned long long* h) {
  read_dev(c, h, ctr(c), sizeof(unsigned long long) * C_NCOUNTERS);
}

// =========================================================== scan ===============
template <class T>
static T scan_excl(sph_ctx* c, const T* in, T* out, int64_t n) {
  if (n <= 0) return T(0);
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  T* sums = reinterpret_cast<T*>(B<char>(c, B_SCAN_TMP, (nb + 2) * sizeof(T)));
  LAUNCH(k_scan_reduce<T>, (int)nb, SCAN_THREADS, 0, in, n, sums);
  LAUNCH(k_scan_blocksums<T>, 1, SCAN_THREADS, 0, sums, nb, sums + nb);
  LAUNCH(k_scan_final<T>, (int)nb, SCAN_THREADS, 0, in, n, sums, out);
  T total;
  read_dev(c, &total, sums + nb, sizeof(T));
  return total;
}

// the same scan leaving its total on the device (no host round trip): returns its address
template <class T>
static const T* scan_excl_dev(sph_ctx* c, const T* in, T* out, int64_t n) {
  int64_t nb = std::max<int64_t>((n + SCAN_TILE - 1) / SCAN_TILE, 1);
  T* sums = reinterpret_cast<T*>(B<char>(c, B_SCAN_TMP, (nb + 2) * sizeof(T)));
  LAUNCH(k_scan_reduce<T>, (int)nb, SCAN_THREADS, 0, in, n, sums);
  LAUNCH(k_scan_blocksums<T>, 1, SCAN_THREADS, 0, sums, nb, sums + nb);
  LAUNCH(k_scan_final<T>, (int)nb, SCAN_THREADS, 0, in, n, sums, out);
  return sums + nb;
}

// =========================================================== kernel attributes ==
// cudaFuncSetAttribute acts on the current device: remember (device, kernel) pairs, so a
// second context on another GPU of the same process raises the limit there too.
static std::mutex g_attr_mu;
static std::set<std::pair<int, const void*>> g_attr_done;
static void ensure_smem_attr(sph_ctx* c, const void* func, int bytes) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  const auto key = std::make_pair(c->device, func);
  if (g_attr_done.count(key)) return;
  CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  g_attr_done.insert(key);
}

// =========================================================== radix sort =========
// hist_ready: B_SORT_HIST already holds every pass's digit counts (k_keys computes them)
static void radix_sort(sph_ctx* c, uint64_t*& keys, uint32_t*& vals, uint64_t*& kalt, uint32_t*& valt,
                       int64_t n, int bits, bool hist_ready = false) {
  if (n <= 1) return;
  int npass = std::max(1, (bits + 7) / 8);
  SPH_REQUIRE(npass <= 8, SPH_E_ARG, "radix sort: more than 64 key bits");
  SPH_REQUIRE(n < (1ll << 30), SPH_E_ARG, "radix sort: n >= 2^30");
  uint32_t* hist = B<uint32_t>(c, B_SORT_HIST, 16 * 256);
  if (!hist_ready) {
    CUDA_TRY(cudaMemsetAsync(hist, 0, 8 * 256 * sizeof(uint32_t), c->stream));
    LAUNCH(k_radix_hist, grid1d(c, n, 256), 256, 0, keys, n, npass, hist);
  }
  uint32_t* gofs = hist + 8 * 256;
  LAUNCH(k_radix_offsets, npass, 256, 0, hist, gofs);
  int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  uint32_t* status = B<uint32_t>(c, B_SORT_STATUS, ntiles * 256);
  uint32_t* tctr = B<uint32_t>(c, B_SORT_CTR, 8);
  ensure_smem_attr(c, (const void*)k_radix_pass, (int)sizeof(RadixSmem));
  CUDA_TRY(cudaMemsetAsync(tctr, 0, 8 * sizeof(uint32_t), c->stream));
  for (int p = 0; p < npass; ++p) {
    CUDA_TRY(cudaMemsetAsync(status, 0, ntiles * 256 * sizeof(uint32_t), c->stream));
    LAUNCH(k_radix_pass, (int)ntiles, RS_THREADS, sizeof(RadixSmem), keys, vals, kalt, valt, n, 8 * p,
           gofs + 256 * p, status, tctr + p);
    std::swap(keys, kalt);
    std::swap(vals, valt);
  }
}

// =========================================================== nodes ==============
static NodeArrays nodes(sph_ctx* c) {
  NodeArrays N;
  N.first = Bget<int>(c, B_N_FIRST);
  N.count = Bget<int>(c, B_N_COUNT);
  N.ijk = Bget<int4>(c, B_N_IJK);
  N.parent = Bget<int>(c, B_N_PARENT);
  N.child = Bget<int>(c, B_N_CHILD);
  N.split = Bget<int>(c, B_N_SPLIT);
  N.hmax = Bget<float>(c, B_N_HMAX);
  N.sortoff = Bget<int64_t>(c, B_N_SORTOFF);
  N.rec = Bget<int4>(c, B_N_REC);
  return N;
}

static void ensure_nodes(sph_ctx* c, int64_t cap) {
  B<int>(c, B_N_FIRST, cap, true);
  B<int>(c, B_N_COUNT, cap, true);
  B<int4>(c, B_N_IJK, cap, true);
  B<int>(c, B_N_PARENT, cap, true);
  B<int>(c, B_N_CHILD, 8 * cap, true);
  B<int>(c, B_N_SPLIT, cap, true);
}

static LevelGeom level_geom(sph_ctx* c) {
  LevelGeom g;
  memset(&g, 0, sizeof(g));
  for (int l = 0; l <= SPH_MAX_DEPTH + 1; ++l)
    for (int k = 0; k < 3; ++k) g.E[l][k] = (float)(c->E0[k] / (double)(1 << l));
  for (int k = 0; k < 3; ++k) {
    g.L[k] = (float)c->cfg.box[k];
    g.ntop[k] = c->ntop[k];
  }
  g.depth = c->depth;
  return g;
}

// largest h the iteration may reach: below half the smallest box edge (minimum image, R19)
static float h_cap(sph_ctx* c) {
  double Lmin = std::min(c->cfg.box[0], std::min(c->cfg.box[1], c->cfg.box[2]));
  return (float)(0.5 * Lmin * (1.0 - 1e-4));
}

static float as_float(unsigned long long b) {
  uint32_t u = (uint32_t)b;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static float3 box3(sph_ctx* c) {
  return make_float3((float)c->cfg.box[0], (float)c->cfg.box[1], (float)c->cfg.box[2]);
}

// =========================================================== build ==============
// a2 + a3: top grid, keys, radix sort, cell-order positions (h from B_HIN or 0).
// Top cell edge >= kappa * max h0 ("larger or equal" to h) and >= TOP_EDGE_HMEAN
// times the mean-density h (Eq. 3 at the mean number density), so that top cells in
// under-dense regions still hold enough particles to fill a warp; the hierarchy below
// splits on occupancy (and on h with the paper's fraction rule, a4). The list walk
// (lists.cuh) handles any h < L/2, so the top grid never has to be rebuilt when h grows.
#define TOP_EDGE_HMEAN 4.0
// Morton levels keyed below the top grid: at least SORT_DEPTH_MIN (C4 uses 8 below its
// 14^3 top cells), and as many more as fit in the same number of 8-bit radix passes; a leaf
// at the deepest keyed level just stays larger (results do not depend on the depth)
#ifndef SORT_DEPTH_MIN
#define SORT_DEPTH_MIN 9
#endif
static void sort_particles(sph_ctx* c, float h0max, bool have_h) {
  DbgTimer _t(c, "sort");
  PhaseTimer _p(c, 3);
  const int64_t n = c->n;
  const double L[3] = {c->cfg.box[0], c->cfg.box[1], c->cfg.box[2]};
  const double V = L[0] * L[1] * L[2];
  const double hmean = cbrt(3.0 * c->cfg.n_ngb * V / (4.0 * M_PI * (double)n));
  const double htop = std::max(TOP_EDGE_HMEAN * hmean, c->cfg.top_edge_factor * (double)h0max) * (1.0 + 1e-6);
  int64_t ntot = 1;
  for (int k = 0; k < 3; ++k) {
    double nk = floor(L[k] / htop);
    nk = std::max(3.0, std::min(nk, 1024.0));
    c->ntop[k] = (int)nk;
    c->E0[k] = L[k] / nk;
    ntot *= (int64_t)nk;
  }
  int top_bits = 0;
  while ((1ll << top_bits) < ntot) ++top_bits;
  const int passes = (top_bits + 3 * SORT_DEPTH_MIN + 7) / 8;
  int depth = std::min(SPH_MAX_DEPTH, (8 * passes - top_bits) / 3);
  depth = std::min(depth, (63 - top_bits) / 3);
  c->depth = depth;
  c->top_bits = top_bits;
  const int kbits = top_bits + 3 * depth;
  c->sort_bits = kbits;
  c->sort_passes = (kbits + 7) / 8;
  uint64_t* k0 = B<uint64_t>(c, B_KEYS0, n);
  uint64_t* k1 = B<uint64_t>(c, B_KEYS1, n);
  uint32_t* v0 = B<uint32_t>(c, B_VALS0, n);
  uint32_t* v1 = B<uint32_t>(c, B_VALS1, n);
  B<uint32_t>(c, B_PERM, n);
  const double sc[3] = {(double)((int64_t)c->ntop[0] << depth) / L[0], (double)((int64_t)c->ntop[1] << depth) / L[1],
                        (double)((int64_t)c->ntop[2] << depth) / L[2]};
  uint32_t* hist = B<uint32_t>(c, B_SORT_HIST, 16 * 256);
  CUDA_TRY(cudaMemsetAsync(hist, 0, 8 * 256 * sizeof(uint32_t), c->stream));
  float4* xc = B<float4>(c, B_XC, n);
  LAUNCH(k_keys, grid1d(c, n, 256), 256, 0, c->xin, have_h ? c->hin : nullptr, n, (float)L[0], (float)L[1],
         (float)L[2], c->ntop[0], c->ntop[1], c->ntop[2], depth, sc[0], sc[1], sc[2], c->sort_passes, k0, v0, xc, hist,
         ctr(c));
  radix_sort(c, k0, v0, k1, v1, n, kbits, true);
  // the sorted keys / permutation: the buffers holding the result take the names KEYS0 and
  // PERM (slot swaps, no copies)
  if (k0 != Bget<uint64_t>(c, B_KEYS0)) std::swap(c->b[B_KEYS0], c->b[B_KEYS1]);
  if (v0 == Bget<uint32_t>(c, B_VALS0)) std::swap(c->b[B_PERM], c->b[B_VALS0]);
  else std::swap(c->b[B_PERM], c->b[B_VALS1]);
  float4* xh = B<float4>(c, B_XH, n);
  // cell-order positions (the pseudo-Verlet reference is copied from them by the first
  // sph_update_cells after this build, not written by every build)
  LAUNCH(k_pack, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, xc, xh);
  c->xref_valid = false;
  c->skin = 0.f;
  // the position checks of k_keys (the sort itself is harmless on invalid input, and so is the
  // level build on its keys) are read with the level build's status: one round trip for both
  c->pos_check = true;
}

static void pos_check(sph_ctx* c, unsigned long long err) {
  c->pos_check = false;
  SPH_REQUIRE(!(err & ERRBIT_NONFINITE), SPH_E_DOMAIN, "non-finite position");
  SPH_REQUIRE(!(err & ERRBIT_XRANGE), SPH_E_DOMAIN, "position outside [0, L)");
}

// a4: the hierarchy from the sorted keys. Split rule: count > split_count and (rule on)
// more than split_fraction of the particles have h < edge/2; with
// use_fraction false the count alone decides (occupancy tree of the cold start).
static void build_nodes(sph_ctx* c, bool use_fraction, bool guess = false, bool guess_all = false) {
  DbgTimer _t(c, "nodes");
  const int64_t n = c->n;
  const uint64_t* keys = Bget<uint64_t>(c, B_KEYS0);
  const float4* xh = Bget<float4>(c, B_XH);
  int* flag = B<int>(c, B_TMPI0, n);
  int* idx = B<int>(c, B_TMPI1, n);
  const int depth = c->depth;
  const int sh = 3 * depth;
  LAUNCH(k_mark_top, grid1d(c, n, 256), 256, 0, keys, n, sh, flag);
  const int64_t ntot = (int64_t)c->ntop[0] * c->ntop[1] * c->ntop[2];
  // the occupied top cells n0 <= min(ntot, n) stay on the device (k_top_counts and
  // k_build_levels read them) when that bound is small; else the count is read first
  const int* n0d = scan_excl_dev<int>(c, flag, idx, n);
  const int64_t n0b = std::min<int64_t>(ntot, n);
  int n0h = -1;
  if (n0b > n / 8) {
    read_dev(c, &n0h, n0d, sizeof(int));
    ensure_nodes(c, std::max<int64_t>(2 * (int64_t)n0h + 1024, n / 8));
  } else {
    ensure_nodes(c, std::max<int64_t>(2 * n0b + 1024, n / 8));
  }
  int* topmap = B<int>(c, B_TOPMAP, ntot);
  CUDA_TRY(cudaMemsetAsync(topmap, 0xff, ntot * sizeof(int), c->stream));
  NodeArrays N = nodes(c);
  LAUNCH(k_write_top, grid1d(c, n, 256), 256, 0, keys, n, sh, flag, idx, c->ntop[0], c->ntop[1], N, topmap);
  LAUNCH(k_top_counts, gridfull(n0h >= 0 ? n0h : n0b, 256), 256, 0, n0d, n, N);
  // the levels in one cooperative launch (k_build_levels); grown and re-run if the nodes
  // outgrow the arrays (they keep their size across builds)
  const LevelGeom g = level_geom(c);
  const float frac = use_fraction ? c->cfg.split_fraction : 0.f;
  int grid = 0;
  {
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_build_levels, LEVEL_THREADS, 0));
    grid = std::max(1, per_sm) * c->num_sms;
  }
  int* lev = B<int>(c, B_N_LEV, SPH_MAX_DEPTH + 12);
  int* part = B<int>(c, B_N_CHBASE, grid);
  for (int attempt = 0;; ++attempt) {
    const int64_t cap = std::min({(int64_t)(c->b[B_N_FIRST].bytes / sizeof(int)),
                                  (int64_t)(c->b[B_N_COUNT].bytes / sizeof(int)),
                                  (int64_t)(c->b[B_N_IJK].bytes / sizeof(int4)),
                                  (int64_t)(c->b[B_N_PARENT].bytes / sizeof(int)),
                                  (int64_t)(c->b[B_N_CHILD].bytes / (8 * sizeof(int))),
                                  (int64_t)(c->b[B_N_SPLIT].bytes / sizeof(int))});
    LevelBuild Lb;
    Lb.lev_off = lev;
    Lb.status = lev + SPH_MAX_DEPTH + 4;
    Lb.bar = reinterpret_cast<unsigned*>(lev + SPH_MAX_DEPTH + 6);
    Lb.part = part;
    Lb.nch = B<int>(c, B_N_NCH, cap);
    Lb.cap = (int)std::min<int64_t>(cap, INT_MAX);
    Lb.presort = lev + SPH_MAX_DEPTH + 8;
    Lb.sort_min_len = c->cfg.sort_min_len;
    Lb.ngroups = lev + SPH_MAX_DEPTH + 9;
    Lb.cmax = c->group_cmax;
    CUDA_TRY(cudaMemsetAsync(lev, 0, (SPH_MAX_DEPTH + 12) * sizeof(int), c->stream));
    N = nodes(c);
    float guess_n = guess ? c->cfg.n_ngb : 0.f;
    int guess_min = guess_all ? -(int)c->cfg.n_ngb : (int)c->cfg.n_ngb;
    float hcap = h_cap(c);
    float4* xh_w = Bget<float4>(c, B_XH);
    const int* n0_arg = n0d;
    void* args[] = {&Lb,  (void*)&xh, (void*)&keys, (void*)&g,  (void*)&depth, &c->cfg.split_count, (void*)&frac,
                    &N,   &guess_n,   &guess_min,   &hcap,      &xh_w,         (void*)&n0_arg};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_build_levels, grid, LEVEL_THREADS, args, 0, c->stream));
    c->launches++;
    // the level offsets and status, and the position checks of the sort, in one round trip
    int hl[SPH_MAX_DEPTH + 10];
    CUDA_TRY(cudaMemcpyAsync(c->hpin, lev, sizeof(hl), cudaMemcpyDeviceToHost, c->stream));
    if (c->pos_check)
      CUDA_TRY(cudaMemcpyAsync(c->hpin + 16, ctr(c) + C_ERR, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    sync(c);
    memcpy(hl, c->hpin, sizeof(hl));
    if (c->pos_check) pos_check(c, c->hpin[16]);
    c->maybe_presort = hl[SPH_MAX_DEPTH + 8] != 0;
    c->n_groups_lev = c->group_cmax > 0 ? hl[SPH_MAX_DEPTH + 9] : -1;
    SPH_REQUIRE(hl[SPH_MAX_DEPTH + 5] != 2, SPH_E_CUDA, "k_build_levels: grid barrier timed out");
    if (hl[SPH_MAX_DEPTH + 5] == 1) {   // node capacity exceeded: grow and run again
      SPH_REQUIRE(attempt < 8, SPH_E_OOM, "node arrays keep overflowing");
      ensure_nodes(c, 2 * cap);
      continue;
    }
    c->lev_off.assign({0, hl[1]});   // [1] = n0, written by k_build_levels
    for (int l = 0; l + 2 < SPH_MAX_DEPTH + 4 && hl[l + 2] > hl[l + 1]; ++l) c->lev_off.push_back(hl[l + 2]);
    break;
  }
  c->n_nodes = c->lev_off.back();
  B<float>(c, B_N_HMAX, c->n_nodes);
  B<int64_t>(c, B_N_SORTOFF, c->n_nodes);
  B<int4>(c, B_N_REC, c->n_nodes);
  N = nodes(c);
  LAUNCH(k_node_rec, gridfull(c->n_nodes, 256), 256, 0, c->n_nodes, N, N.rec);
}

// a6: the 13 presorted directions of every leaf longer than sort_min_len
static void build_sorted(sph_ctx* c) {
  DbgTimer _t(c, "sorted lists");
  const int nn = c->n_nodes;
  if (!c->maybe_presort) {   // no leaf qualifies (k_build_levels): no lists, no scan
    c->n_sorted = 0;
    CUDA_TRY(cudaMemsetAsync(Bget<int64_t>(c, B_N_SORTOFF), 0xff, nn * sizeof(int64_t), c->stream));
    return;
  }
  int64_t* sz = B<int64_t>(c, B_TMPL0, nn);
  int64_t* sc = B<int64_t>(c, B_TMPL1, nn);
  NodeArrays N = nodes(c);
  LAUNCH(k_sort_sizes, gridfull(nn, 256), 256, 0, nn, N, c->cfg.sort_min_len, sz);
  c->n_sorted = scan_excl<int64_t>(c, sz, sc, nn);
  LAUNCH(k_sort_offsets, gridfull(nn, 256), 256, 0, nn, sz, sc, N);
  if (c->n_sorted == 0) return;
  SortEntry* sorted = B<SortEntry>(c, B_SORTED, c->n_sorted);
  const LevelGeom g = level_geom(c);
  const float4* xh = Bget<float4>(c, B_XH);
  LAUNCH(k_sort_leaf_warp, gridfull((int64_t)nn * 32, 256), 256, 0, nn, xh, N, g, sorted);
  const int smem = SORT_BLOCK_MAX * (8 + 4);
  ensure_smem_attr(c, (const void*)k_sort_leaf_block, smem);
  LAUNCH(k_sort_leaf_block, nn, 512, smem, nn, xh, N, g, sorted);
}

static void build_groups(sph_ctx* c) {
  const int nn = c->n_nodes;
  int* nchunk = B<int>(c, B_TMPI0, nn);
  int* cscan = B<int>(c, B_TMPI1, nn);
  NodeArrays N = nodes(c);
  const int cmax = c->group_cmax;
  LAUNCH(k_group_count, gridfull(nn, 256), 256, 0, nn, N, cmax, nchunk);
  if (c->n_groups_lev >= 0) {   // counted by the level build: the offsets stay on the device
    scan_excl_dev<int>(c, nchunk, cscan, nn);
    c->n_groups = c->n_groups_lev;
  } else {
    c->n_groups = scan_excl<int>(c, nchunk, cscan, nn);
  }
  int4* groups = B<int4>(c, B_GROUPS, c->n_groups);
  LAUNCH(k_group_write, gridfull(nn, 256), 256, 0, nn, N, cmax, cscan, groups);
}

// dynamic shared memory of the walk (WALK_WARPS x WalkSmem > the 48 KB static limit)
static int walk_smem(sph_ctx* c) {
  const int bytes = WALK_WARPS * (int)sizeof(WalkSmem);
  ensure_smem_attr(c, (const void*)k_walk<MODE_NB>, bytes);
  ensure_smem_attr(c, (const void*)k_walk<MODE_FILL>, bytes);
  return bytes;
}

static WalkParams walk_params(sph_ctx* c, const float* reach) {
  WalkParams P;
  memset(&P, 0, sizeof(P));
  // [0] neighbour-list walks since the build, [1] interaction-list walks of the last density call
  if (c->cfg.flags & SPH_F_COUNT_CANDIDATES) P.raw_out = Bget<unsigned long long>(c, B_WALKRAW);
  P.groups = Bget<int4>(c, B_GROUPS);
  P.xh = Bget<float4>(c, B_XH);
  P.reach = reach;
  P.perm = Bget<uint32_t>(c, B_PERM);
  P.n_own = c->n_own;
  P.tgt = Bget<uint8_t>(c, B_TGT);
  P.N = nodes(c);
  P.g = level_geom(c);
  P.topmap = Bget<int>(c, B_TOPMAP);
  P.sorted = Bget<SortEntry>(c, B_SORTED);
  P.any_sorted = c->n_sorted > 0;
  float Lmax = (float)std::max(c->cfg.box[0], std::max(c->cfg.box[1], c->cfg.box[2]));
  P.slack = 4e-7f * Lmax + c->skin;   // + the drift since the cells were sorted (sph_update_cells)
  P.ctr = ctr(c);
  return P;
}

// NB walk: per target (the owned, active particles if tsel_val < 0, else those in state
// tsel_val, over only the groups the last solve listed) the squared distances
// r^2 < h_build^2 (lists.cuh, MODE_NB), with the h iteration fused into the walk's epilogue
// and the re-walks of its particles in the same warp; overflows and leftovers are counted
// on the device (B_HCTR), read once per host round.
static float solve_margin(sph_ctx* c) { return std::max(c->cfg.h_margin, c->regrow_margin); }

static void nb_walk(sph_ctx* c, int tsel_val, int64_t n_regrow = 0) {
  DbgTimer _t(c, "neighbour lists + h solve");
  const int64_t n = c->n;
  WalkParams P = walk_params(c, Bget<float>(c, B_HB));
  P.nsel = c->n_groups;
  const int ng = c->n_groups;
  int* rgl = B<int>(c, B_RGL, 2 * (int64_t)std::max(ng, 1));
  int* rgc = B<int>(c, B_RGCNT, 2);
  if (tsel_val >= 0) {
    P.tsel = Bget<uint8_t>(c, B_STATE);
    P.tsel_val = (uint8_t)tsel_val;
    if (tsel_val == HS_REGROW && c->rg_valid) {
      // only the groups the last solve left with re-walking particles (at most one per particle)
      P.sel = rgl + (int64_t)c->rg_cur * ng;
      P.nsel_dev = rgc + c->rg_cur;
      P.nsel = (int)std::min<int64_t>(ng, n_regrow);
    }
  }
  // this walk's solve appends its re-walk groups to the other list
  const int nxt = P.nsel_dev ? 1 - c->rg_cur : c->rg_cur;
  CUDA_TRY(cudaMemsetAsync(rgc + nxt, 0, sizeof(int), c->stream));
  P.rg_out = rgl + (int64_t)nxt * ng;
  P.rg_cnt = rgc + nxt;
  c->rg_cur = nxt;
  c->rg_valid = true;
  P.K = c->nb_k;
  P.nb_entries = Bget<unsigned long long>(c, B_NBENT);
  P.nb_r2 = B<float>(c, B_NBR2, (size_t)n * c->nb_k);
  P.nb_cnt = B<int>(c, B_NBCNT, n);
  P.solve = 1;
  P.hb_w = Bget<float>(c, B_HB);
  P.lo = Bget<float>(c, B_HLO);
  P.hi = Bget<float>(c, B_HHI);
  P.state = Bget<uint8_t>(c, B_STATE);
  P.shrunk = Bget<uint8_t>(c, B_SHRUNK);
  P.ovf_cnt = B<int64_t>(c, B_OVFC, n);
  P.ovf_off_w = Bget<int64_t>(c, B_NBOFF);
  P.hc = B<unsigned long long>(c, B_HCTR, HC_N);
  P.n_t = c->cfg.n_ngb;
  P.tol = c->cfg.n_ngb_tol;
  P.margin = solve_margin(c);
  P.hcap = h_cap(c);
  P.max_iter = c->cfg.max_h_iter;
  {
    PhaseTimer _p(c, 0);
    LAUNCH(k_walk<MODE_NB>, gridfull(P.nsel, WALK_WARPS), WALK_WARPS * 32, walk_smem(c), P);
  }
  c->walk_launches++;
}

// per-round counters (HC_EVALS accumulates over the rounds of a call: zeroed by hctr_zero)
static void hctr_reset(sph_ctx* c) {
  CUDA_TRY(cudaMemsetAsync(B<unsigned long long>(c, B_HCTR, HC_N), 0, HC_EVALS * sizeof(unsigned long long),
                           c->stream));
}
static void hctr_zero(sph_ctx* c) {
  CUDA_TRY(cudaMemsetAsync(B<unsigned long long>(c, B_HCTR, HC_N), 0, HC_N * sizeof(unsigned long long), c->stream));
}

// Particles in state HS_OVF (a repeat overflow): exactly sized lists in the overflow pool
// (contiguous per particle), recorded by a second NB walk of their groups.
static void nb_pool(sph_ctx* c) {
  DbgTimer _t(c, "neighbour lists (pool)");
  const int64_t n = c->n;
  int64_t* oc = Bget<int64_t>(c, B_OVFC);
  int64_t* os = B<int64_t>(c, B_TMPL1, n);
  int64_t* ooff = Bget<int64_t>(c, B_NBOFF);
  uint8_t* state = Bget<uint8_t>(c, B_STATE);
  const int64_t tot = scan_excl<int64_t>(c, oc, os, n);
  if (tot == 0) return;
  const int64_t base = c->ovf_used;
  float* pool = B<float>(c, B_NBOVF, base + tot, true);
  c->ovf_used = base + tot;
  LAUNCH(k_ovf_offsets, grid1d(c, n, 256), 256, 0, n, oc, os, base, ooff);
  {
    // the pool particles' indices, appended to the list k_hsolve_pool walks
    int* pf = B<int>(c, B_TMPI0, n);
    int* ps = B<int>(c, B_TMPI1, n);
    LAUNCH(k_flag_pos64, grid1d(c, n, 256), 256, 0, oc, n, pf);
    const int np = scan_excl<int>(c, pf, ps, n);
    int32_t* idx = B<int32_t>(c, B_OVFIDX, c->n_ovfidx + np, true);
    LAUNCH(k_compact_append, grid1d(c, n, 256), 256, 0, pf, ps, n, idx + c->n_ovfidx);
    c->n_ovfidx += np;
  }
  WalkParams Q = walk_params(c, Bget<float>(c, B_HB));
  Q.nsel = c->n_groups;
  Q.tsel = state;
  Q.tsel_val = HS_OVF;
  Q.K = c->nb_k;
  Q.nb_cnt = Bget<int>(c, B_NBCNT);
  Q.ovf = pool;
  Q.ovf_off = ooff;
  Q.nb_entries = Bget<unsigned long long>(c, B_NBENT);
  {
    PhaseTimer _p(c, 0);
    LAUNCH(k_walk<MODE_NB>, gridfull(Q.nsel, WALK_WARPS), WALK_WARPS * 32, walk_smem(c), Q);
  }
  c->walk_launches++;
  LAUNCH(k_state_swap, grid1d(c, n, 256), 256, 0, state, n, (uint8_t)HS_OVF, (uint8_t)HS_ACTIVE);
  CUDA_TRY(cudaMemsetAsync(oc, 0, n * sizeof(int64_t), c->stream));
  DBG("neighbour lists: %lld entries in the overflow pool\n", (long long)tot);
}

// UNION walk: per group the sources within reach max(h_i, h_j) of at least one target, with
// h from `reach` (lists.cuh). One pass into fixed-capacity slabs (ucap entries per group);
// groups beyond it are walked again into exactly sized space after the slabs.
static void build_union(sph_ctx* c, const float* reach) {
  DbgTimer _t(c, "interaction lists");
  const int ng = c->n_groups;
  if (ng == 0) return;
  // node max of the reach (the walk's bound for sources with a large h); the top cells' maxima
  // give the global max, read by the walk
  ctr_reset(c);
  LAUNCH(k_node_hmax, gridfull((int64_t)c->n_nodes * 32, 256), 256, 0, c->n_nodes, nodes(c), reach, ctr(c));
  unsigned long long h[C_NCOUNTERS];
  const int cap = c->ucap;
  WalkParams P = walk_params(c, reach);
  if (P.raw_out) {
    P.raw_out += 1;
    CUDA_TRY(cudaMemsetAsync(P.raw_out, 0, sizeof(unsigned long long), c->stream));
  }
  P.reach_max_bits = ctr(c) + C_HMAXBITS;
  P.reach_xhw = c->n == c->n_own && reach == Bget<float>(c, B_HRCH);   // k_reach_owned copied xh.w for all
  P.nsel = ng;
  P.off = B<int64_t>(c, B_GOFF, ng);
  P.len = B<int>(c, B_GLEN, ng);
  P.ucap = cap;
  const int64_t slab = (int64_t)ng * cap;
  P.out = B<uint32_t>(c, B_LIST, slab);
  LAUNCH(k_slab_offsets, gridfull(ng, 256), 256, 0, ng, cap, P.off);
  {
    PhaseTimer _p(c, 2);
    LAUNCH(k_walk<MODE_FILL>, gridfull(ng, WALK_WARPS), WALK_WARPS * 32, walk_smem(c), P);
  }
  int* flag = B<int>(c, B_GFLAG, ng);
  int* scan = B<int>(c, B_TMPI1, ng);
  LAUNCH(k_union_overflow, gridfull(ng, 256), 256, 0, ng, P.len, cap, flag);
  const int no = scan_excl<int>(c, flag, scan, ng);
  int64_t total = slab;
  if (no > 0) {
    int* sel = B<int>(c, B_GSEL, no);
    LAUNCH(k_compact_idx, grid1d(c, ng, 256), 256, 0, flag, scan, (int64_t)ng, sel);
    int64_t* l64 = B<int64_t>(c, B_TMPL0, no);
    int64_t* lscan = B<int64_t>(c, B_TMPL1, no);
    LAUNCH(k_gather_len, gridfull(no, 256), 256, 0, no, sel, P.len, l64);
    const int64_t extra = scan_excl<int64_t>(c, l64, lscan, no);
    P.out = B<uint32_t>(c, B_LIST, slab + extra, true);
    total = slab + extra;
    LAUNCH(k_set_offsets, gridfull(no, 256), 256, 0, no, sel, lscan, slab, P.off);
    P.nsel = no;
    P.sel = sel;
    P.ucap = INT32_MAX;
    P.check = 1;
    PhaseTimer _p(c, 2);
    LAUNCH(k_walk<MODE_FILL>, gridfull(no, WALK_WARPS), WALK_WARPS * 32, walk_smem(c), P);
  }
  c->pool = total;
  if (dbg_on()) {
    ctr_read(c, h);
    std::vector<int> hl(ng);
    CUDA_TRY(cudaMemcpyAsync(hl.data(), P.len, ng * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    int64_t ent = 0;
    for (int v : hl) ent += v;
    std::sort(hl.begin(), hl.end());
    DBG("interaction lists: %d groups, %lld entries (%.1f per group; p50 %d p99 %d max %d), %d beyond the slab; "
        "raw sources %llu (max %llu per group)\n", ng, (long long)ent, (double)ent / ng, hl[ng / 2],
        hl[(int)(0.99 * (ng - 1))], hl[ng - 1], no, h[C_TMP2], h[C_TMP0]);
  }
}

static GroupLists group_lists(sph_ctx* c) {
  GroupLists G;
  G.groups = Bget<int4>(c, B_GROUPS);
  G.off = Bget<int64_t>(c, B_GOFF);
  G.len = Bget<int>(c, B_GLEN);
  G.list = Bget<uint32_t>(c, B_LIST);
  G.ngroups = c->n_groups;
  return G;
}

// =========================================================== inputs =============
// page-locked host memory (cudaMallocHost / cudaHostRegister): copies to it are asynchronous
static bool is_pinned_host_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// device view of a caller input array: the pointer itself, or a staged copy
template <class T>
static const T* dev_in(sph_ctx* c, const T* p, size_t count, int stage_id, bool force_copy = false) {
  if (is_device_ptr(p) && !force_copy) return p;
  T* d = B<T>(c, stage_id, count);
  CUDA_TRY(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyDefault, c->stream));
  return d;
}

struct OutMap {
  void* user;
  void* dev;
  size_t bytes;
};
template <class T>
static T* dev_out(sph_ctx* c, T* p, size_t count, int stage_id, std::vector<OutMap>& maps) {
  if (!p) return nullptr;
  if (is_device_ptr(p)) return p;
  T* d = B<T>(c, stage_id, count);
  maps.push_back(OutMap{p, d, count * sizeof(T)});
  return d;
}
static void flush_out(sph_ctx* c, std::vector<OutMap>& maps, cudaEvent_t done) {
  for (auto& m : maps)
    CUDA_TRY(cudaMemcpyAsync(m.user, m.dev, m.bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaEventRecord(done, c->stream));
  if (!maps.empty()) sync(c);
}


// =========================================================== API ================
#define API_BEGIN(ctx)                                                              \
  if (!(ctx)) return SPH_E_ARG;                                                     \
  sph_ctx* c = (ctx);                                                               \
  c->err.clear();                                                                   \
  try {                                                                             \
    CUDA_TRY(cudaSetDevice(c->device));
#define API_END                                                                     \
  }                                                                                 \
  catch (const SphError& e) {                                                       \
    c->err = e.msg;                                                                 \
    if (e.status == SPH_E_CUDA) cudaGetLastError();                                 \
    return e.status;                                                                \
  }                                                                                 \
  catch (const std::exception& e) {                                                 \
    c->err = e.what();                                                              \
    return SPH_E_CUDA;                                                              \
  }

extern "C" {

void sph_config_default(sph_config* cfg, double lx, double ly, double lz) {
  memset(cfg, 0, sizeof(*cfg));
  cfg->abi_version = SPH_ABI_VERSION;
  cfg->box[0] = lx;
  cfg->box[1] = ly;
  cfg->box[2] = lz;
  cfg->gamma = 5.0f / 3.0f;
  cfg->n_ngb = 48.0f;
  cfg->n_ngb_tol = 1e-4f;
  cfg->max_h_iter = 64;
  cfg->alpha = 0.8f;
  cfg->balsara_eps = 1e-4f;
  cfg->split_count = 300;
  cfg->split_fraction = 0.875f;
  cfg->top_edge_factor = 1.0f;
  cfg->h_margin = 1.1f;
  cfg->sort_min_len = 64;
  cfg->flags = SPH_F_SYNC;
  cfg->rank = 0;
  cfg->nranks = 1;
  cfg->slab_lo = 0.0;
  cfg->slab_hi = lx;
  cfg->halo_width = 0.0;
}

const char* sph_status_string(int s) {
  switch (s) {
    case SPH_OK: return "SPH_OK";
    case SPH_E_ARG: return "SPH_E_ARG: invalid argument or configuration";
    case SPH_E_DOMAIN: return "SPH_E_DOMAIN: input outside the method's domain";
    case SPH_E_STATE: return "SPH_E_STATE: calls out of order";
    case SPH_E_NOCONV: return "SPH_E_NOCONV: h iteration did not converge";
    case SPH_E_CUDA: return "SPH_E_CUDA: CUDA error";
    case SPH_E_NCCL: return "SPH_E_NCCL: NCCL error";
    case SPH_E_OOM: return "SPH_E_OOM: out of device memory";
    default: return "unknown sph_status";
  }
}

const char* sph_last_error(const sph_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t sph_kernel_launches(const sph_ctx* c) { return c ? c->launches : 0; }

static bool cfg_ok(const sph_config* f, std::string& why) {
  if (f->abi_version != SPH_ABI_VERSION) { why = "abi_version mismatch"; return false; }
  for (int k = 0; k < 3; ++k)
    if (!(f->box[k] > 0.0)) { why = "box <= 0"; return false; }
  if (!(f->gamma > 1.f)) { why = "gamma <= 1"; return false; }
  if (!(f->alpha >= 0.f)) { why = "alpha < 0"; return false; }
  if (!(f->n_ngb > 32.f / 3.f)) { why = "n_ngb <= 32/3 (the self term alone)"; return false; }
  if (!(f->n_ngb_tol > 0.f)) { why = "n_ngb_tol <= 0"; return false; }
  if (!(f->top_edge_factor >= 1.f)) { why = "top_edge_factor < 1"; return false; }
  if (!(f->h_margin >= 1.f)) { why = "h_margin < 1"; return false; }
  if (f->sort_min_len < 0) { why = "sort_min_len < 0"; return false; }
  if (!(f->split_fraction >= 0.f && f->split_fraction < 1.f)) { why = "split_fraction outside [0,1)"; return false; }
  if (f->split_count < 1) { why = "split_count < 1"; return false; }
  if (f->max_h_iter < 1) { why = "max_h_iter < 1"; return false; }
  if (f->row_cap < 0 || f->list_cap < 0 || f->cold_margin < 0.f || f->group_container < -1) {
    why = "negative capacity or margin";
    return false;
  }
  if (f->nranks < 1 || f->rank < 0 || f->rank >= f->nranks) { why = "bad rank/nranks"; return false; }
  return true;
}

int sph_create(const sph_config* cfg, int dev, void* stream, sph_ctx** out) {
  if (!out) return SPH_E_ARG;
  *out = nullptr;
  if (!cfg) return SPH_E_ARG;
  std::string why;
  if (!cfg_ok(cfg, why)) return SPH_E_ARG;
  sph_ctx* c = new sph_ctx();
  c->cfg = *cfg;
  c->device = dev;
  try {
    CUDA_TRY(cudaSetDevice(dev));
    int ns = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&ns, cudaDevAttrMultiProcessorCount, dev));
    c->num_sms = ns;
    CUDA_TRY(cudaMallocHost((void**)&c->hpin, 64 * sizeof(unsigned long long)));
    if (stream) {
      c->stream = (cudaStream_t)stream;
    } else {
      // a blocking stream: ordered after work on the legacy default stream (e.g. torch's
      // tensors produced there), so a caller that passes no stream gets no race
      CUDA_TRY(cudaStreamCreate(&c->stream));
      c->own_stream = true;
    }
    for (int i = 0; i < 12; ++i) CUDA_TRY(cudaEventCreate(&c->ev[i]));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
    for (int i = 0; i < 6; ++i) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_side[i], cudaEventDisableTiming));
    float dirs[14][3];
    for (int d = 0; d < 13; ++d) {
      const int k = d + 14;
      const double ox = off_x(k), oy = off_y(k), oz = off_z(k);
      const double inv = 1.0 / sqrt(ox * ox + oy * oy + oz * oz);
      dirs[d][0] = (float)(ox * inv);
      dirs[d][1] = (float)(oy * inv);
      dirs[d][2] = (float)(oz * inv);
    }
    dirs[13][0] = dirs[13][1] = dirs[13][2] = 0.f;
    CUDA_TRY(cudaMemcpyToSymbol(c_dirs, dirs, sizeof(dirs)));
    c->ev_ok = true;
    // capacities and tuning from the config (include/sph.h); defaults otherwise
    if (cfg->cold_margin > 0.f) c->cold_margin = cfg->cold_margin;
    if (cfg->list_cap > 0) c->ucap = cfg->list_cap;
    if (cfg->group_container != 0) c->group_cmax = cfg->group_container < 0 ? 0 : cfg->group_container;
  } catch (const SphError& e) {
    if (c->hpin) cudaFreeHost(c->hpin);
    delete c;
    return e.status;
  }
  *out = c;
  return SPH_OK;
}

int sph_destroy(sph_ctx* c) {
  if (!c) return SPH_E_ARG;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (int i = 0; i < B_COUNT; ++i) dev_free(c, c->b[i].p);
  if (c->hpin) cudaFreeHost(c->hpin);
  for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
  for (void* p : c->ipc_own) cudaFree(p);
  for (cudaEvent_t e : c->ipc_ev) cudaEventDestroy(e);
  if (c->ev_ok) {
    for (int i = 0; i < 12; ++i) cudaEventDestroy(c->ev[i]);
    for (int i = 0; i < 6; ++i) cudaEventDestroy(c->ev_side[i]);
    cudaStreamDestroy(c->stream2);
  }
  for (auto& t : c->timed) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->comm) nccl().CommDestroy((ncclComm_t)c->comm);
  delete c;
  return SPH_OK;
}

int sph_set_allocator(sph_ctx* c, void* (*alloc)(size_t, void*, void*), void (*release)(void*, void*, void*),
                      void* user) {
  if (!c) return SPH_E_ARG;
  if ((alloc == nullptr) != (release == nullptr)) return SPH_E_ARG;
  for (int i = 0; i < B_COUNT; ++i)
    if (c->b[i].p) return SPH_E_STATE;
  c->ualloc = alloc;
  c->urelease = release;
  c->uuser = user;
  return SPH_OK;
}

static bool stage_vmu(sph_ctx* c, const float* v, const float* m, const float* u, const float* dv[3]);

int sph_build_cells(sph_ctx* ctx, int64_t n, const float* x, const float* h0) {
  return sph_build_cells_halo(ctx, n, 0, x, h0);
}

// positions in, validated; h0 (optional) in, validated; returns whether a guess is needed
// Positions and h0 for this call: device arrays are used in place (they are consumed inside
// the call), host arrays copied in. h0 is validated here (its largest value sets the top grid);
// the positions are validated by k_keys (or k_validate_x, validate_x = true). Returns whether
// a guess is needed.
static bool load_inputs(sph_ctx* c, const float* x, const float* h0, float* h0max, bool validate_x = false) {
  const int64_t n = c->n;
  if (is_device_ptr(x)) {
    c->xin = x;
  } else {
    float* xd = B<float>(c, B_XIN, 3 * n);
    CUDA_TRY(cudaMemcpyAsync(xd, x, 3 * n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    c->xin = xd;
  }
  ctr_reset(c);
  if (validate_x)
    LAUNCH(k_validate_x, grid1d(c, n, 256), 256, 0, c->xin, n, (float)c->cfg.box[0], (float)c->cfg.box[1],
           (float)c->cfg.box[2], ctr(c));
  c->hin = nullptr;
  unsigned long long hc[C_NCOUNTERS];
  if (h0) {
    if (is_device_ptr(h0)) {
      c->hin = h0;
    } else {
      float* hd = B<float>(c, B_HIN, n);
      CUDA_TRY(cudaMemcpyAsync(hd, h0, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      c->hin = hd;
    }
    LAUNCH(k_hrange, grid1d(c, n, 256), 256, 0, c->hin, n, ctr(c));
  }
  if (h0 || validate_x) {
    ctr_read(c, hc);
    SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_NONFINITE), SPH_E_DOMAIN, "non-finite position");
    SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_XRANGE), SPH_E_DOMAIN, "position outside [0, L)");
    SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_H), SPH_E_DOMAIN, "h0 negative or non-finite");
  }
  *h0max = h0 ? as_float(hc[C_HMAXBITS]) : 0.f;
  SPH_REQUIRE(*h0max < h_cap(c), SPH_E_DOMAIN,
              "h0 >= min(L)/2: the minimum-image convention needs h < L/2 (h0 max = " + std::to_string(*h0max) + ")");
  if (h0) ctr_reset(c);
  return !h0 || hc[C_TMP0] > 0;
}

int sph_build_cells_halo(sph_ctx* ctx, int64_t n_own, int64_t n_halo, const float* x, const float* h0) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n_own > 0 && n_halo >= 0 && x, SPH_E_ARG, "n_own <= 0, n_halo < 0 or x == NULL");
  SPH_REQUIRE(!c->has_active || (h0 && c->n_active_for == n_own), SPH_E_ARG,
              "an active mask (sph_set_active) needs h0 (the inactive particles' h) and n_own particles");
  const int64_t n = n_own + n_halo;
  SPH_REQUIRE(n <= (1ll << SPH_IDX_BITS), SPH_E_ARG, "n > 2^27 particles in one context");
  c->n = n;
  c->n_own = n_own;
  c->state = 0;
  c->force_lists = false;
  if (c->cfg.row_cap > 0) {
    c->nb_k = std::max(4, c->cfg.row_cap & ~3);
  } else if (n != c->nb_k_for) {
    // neighbour-list slab: up to 1024 entries per particle, within 40% of the free device
    // memory (cold-start lists hold ~90 entries; longer ones shrink or go to the pool);
    // sized once per particle count (cudaMemGetInfo stalls the host)
    size_t fr = 0, tot = 0;
    CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    const size_t have = fr + c->b[B_NBR2].bytes;   // the slab of a previous build is reused
    c->nb_k = (int)std::max<int64_t>(64, std::min<int64_t>(1024, (int64_t)(0.4 * (double)have / (4.0 * (double)n))));
    c->nb_k &= ~3;   // rows of K floats stay 16-byte aligned (float4 reads in the h sums)
    c->nb_k_for = n;
  }
  c->pool = 0;
  c->list_rebuilds = 0;
  // side-stream work of an earlier sph_density that returned early must not overlap the
  // staging buffers this build writes
  if (c->ev_ok) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_side[5], 0));
  CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
  phase_reset(c);
  CUDA_TRY(cudaMemsetAsync(B<unsigned long long>(c, B_NBENT, 1), 0, sizeof(unsigned long long), c->stream));
  float h0max = 0.f;
  const bool need_guess = load_inputs(c, x, h0, &h0max);
  if (c->pre_pending) {   // sph_step: v, m, u up on the side stream behind x, during the build
    const float* dv[3];
    c->pre_side = stage_vmu(c, c->pre_in[0], c->pre_in[1], c->pre_in[2], dv);
    for (int k = 0; k < 3; ++k) c->pre_dev[k] = dv[k];
    c->pre_pending = false;
    c->pre_ready = true;
  }
  // a2 + a3: one sort for the whole evaluation
  sort_particles(c, h0max, h0 != nullptr);
  // a4: the hierarchy; the cold start guesses h from the occupancy of the count-rule tree
  const bool frac = c->cfg.split_fraction > 0.f;
  // (the leaves write the guess as the level build decides them: k_build_levels)
  build_nodes(c, frac && !need_guess, need_guess, need_guess && h0 == nullptr);
  float margin = c->cfg.h_margin;
  if (need_guess) {
    // the guess is off by up to ~2x either way (C4 p1/p99 0.68/1.88): record at 1.2x the
    // guess; particles whose root lies beyond it are re-walked in the same warp (lists.cuh)
    margin = c->cold_margin;
    if (frac) build_nodes(c, true);     // the paper's split rule needs h
  }
  c->cold = need_guess;
  c->cells_reused = false;
  // a6 + groups + density lists for h_build = h * margin
  build_sorted(c);
  build_groups(c);
  {
    float* hb = B<float>(c, B_HB, n);
    B<float>(c, B_HLO, n);
    B<float>(c, B_HHI, n);
    B<float>(c, B_HRCH, n);
    B<uint8_t>(c, B_STATE, n);
    CUDA_TRY(cudaMemsetAsync(B<int64_t>(c, B_NBOFF, n), 0xff, n * sizeof(int64_t), c->stream));
    CUDA_TRY(cudaMemsetAsync(B<uint8_t>(c, B_SHRUNK, n), 0, n, c->stream));
    CUDA_TRY(cudaMemsetAsync(B<int64_t>(c, B_OVFC, n), 0, n * sizeof(int64_t), c->stream));
    B<float>(c, B_NBOVF, 1);
    c->ovf_used = 0;
    c->n_ovfidx = 0;
    // targets: owned and active (sph_set_active); everything else is a source only
    LAUNCH(k_make_tgt, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, c->n_own,
           c->has_active ? Bget<uint8_t>(c, B_ACTIVE) : (const uint8_t*)nullptr, B<uint8_t>(c, B_TGT, n));
    LAUNCH(k_init_iter, grid1d(c, n, 256), 256, 0, Bget<uint8_t>(c, B_TGT), n, Bget<float4>(c, B_XH),
           margin, h_cap(c), Bget<uint8_t>(c, B_STATE), hb, Bget<float>(c, B_HLO), Bget<float>(c, B_HHI));
  }
  // neighbour lists of the h iteration: r^2 < h_build^2 per particle
  hctr_zero(c);
  CUDA_TRY(cudaMemsetAsync(B<unsigned long long>(c, B_WALKRAW, 2), 0, 2 * sizeof(unsigned long long), c->stream));
#ifdef SPH_WALK_STATS
  {
    unsigned long long z[8][5] = {};
    CUDA_TRY(cudaMemcpyToSymbolAsync(g_walkstats, z, sizeof(z), 0, cudaMemcpyHostToDevice, c->stream));
  }
#endif
  nb_walk(c, -1);
  c->state = 1;
  CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
  // inside sph_step the density call's first counter read is the next round trip
  if (!c->in_step) sync(c);
#ifdef SPH_WALK_STATS
  {
    unsigned long long z[8][5];
    CUDA_TRY(cudaMemcpyFromSymbol(z, g_walkstats, sizeof(z)));
    for (int p = 0; p < 8; ++p)
      if (z[p][0])
        fprintf(stderr, "[walkstats] pass %d: warp-passes %llu active lanes %llu survivors %llu recorded %llu chunks %llu\n",
                p, z[p][0], z[p][1], z[p][2], z[p][3], z[p][4]);
  }
#endif
  DBG("build: n %lld top %dx%dx%d depth %d levels %zu nodes %d groups %d sorted %lld list %lld\n", (long long)n,
      c->ntop[0], c->ntop[1], c->ntop[2], c->depth, c->lev_off.size() - 1, c->n_nodes, c->n_groups,
      (long long)c->n_sorted, (long long)c->pool);
  API_END
  return SPH_OK;
}

static void fill_struct_stats(sph_ctx* c, sph_stats* st) {
  st->n_levels = (int)c->lev_off.size() - 1;
  st->n_cells = c->n_nodes;
  st->n_leaves = c->n_groups;
  st->n_pair_slots = c->pool;
  st->n_rebuilds = c->list_rebuilds;
}

// v, m, u of host arrays copied on the side stream (device arrays used in place): dv = their
// device views; returns whether a side-stream copy was issued (joined by ev_side[1])
static bool stage_vmu(sph_ctx* c, const float* v, const float* m, const float* u, const float* dv[3]) {
  const int64_t n = c->n;
  const float* in[3] = {v, m, u};
  const int ids[3] = {B_VIN, B_MIN, B_UIN};
  const size_t cnt[3] = {(size_t)(3 * n), (size_t)n, (size_t)n};
  bool side = false;
  for (int k = 0; k < 3; ++k) {
    dv[k] = in[k];
    if (is_device_ptr(in[k])) continue;
    if (!side) {
      CUDA_TRY(cudaEventRecord(c->ev_side[0], c->stream));   // staging buffers free to overwrite
      CUDA_TRY(cudaStreamWaitEvent(c->stream2, c->ev_side[0], 0));
      side = true;
    }
    float* d = B<float>(c, ids[k], cnt[k]);
    CUDA_TRY(cudaMemcpyAsync(d, in[k], cnt[k] * sizeof(float), cudaMemcpyHostToDevice, c->stream2));
    dv[k] = d;
  }
  if (side) CUDA_TRY(cudaEventRecord(c->ev_side[1], c->stream2));
  return side;
}

int sph_density(sph_ctx* ctx, const float* v, const float* m, const float* u, float* h_out, float* rho_out,
                float* omega_out, int32_t* n_nbr_out, float* div_out, float* curl_out, sph_stats* st) {
  API_BEGIN(ctx)
  if (c->has_active) {   // inactive entries are left as they are: only device outputs can be
    const void* outs[6] = {h_out, rho_out, omega_out, n_nbr_out, div_out, curl_out};
    for (const void* o : outs)
      SPH_REQUIRE(!o || is_device_ptr(o), SPH_E_ARG, "with an active mask the outputs must be device arrays");
  }
  SPH_REQUIRE(c->state >= 1, SPH_E_STATE, "sph_density before sph_build_cells");
  SPH_REQUIRE(v && m && u && h_out && rho_out, SPH_E_ARG, "required pointer is NULL");
  const int64_t n = c->n;
  CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
  // v, m, u are first needed after the h iteration: host arrays are copied on the side
  // stream while the rounds run (joined before validation)
  const float* vd = v;
  const float* md = m;
  const float* ud = u;
  bool side = false;
  if (c->pre_ready && c->pre_in[0] == v && c->pre_in[1] == m && c->pre_in[2] == u) {
    // staged by sph_step before the build
    vd = c->pre_dev[0];
    md = c->pre_dev[1];
    ud = c->pre_dev[2];
    side = c->pre_side;
    c->pre_ready = false;
  } else {
    c->pre_ready = false;
    const float* dv[3];
    side = stage_vmu(c, v, m, u, dv);
    vd = dv[0];
    md = dv[1];
    ud = dv[2];
  }
  // v, m, u checked and gathered into cell order on the side stream (behind their copies),
  // concurrently with the h rounds and the union walk; joined before the density kernel
  float4* vm = B<float4>(c, B_VM, n);
  float* uc = B<float>(c, B_U, n);
  unsigned long long* verr = B<unsigned long long>(c, B_VERR, C_NCOUNTERS);
  float4* vmc = B<float4>(c, B_XC, n);   // caller-order {v, m} (the positions' staging is free again)
  CUDA_TRY(cudaEventRecord(c->ev_side[4], c->stream));   // the caller's device arrays, perm
  CUDA_TRY(cudaStreamWaitEvent(c->stream2, c->ev_side[4], 0));
  CUDA_TRY(cudaMemsetAsync(verr, 0, C_NCOUNTERS * sizeof(unsigned long long), c->stream2));
  {
    PhaseTimer _p(c, 3, c->stream2);   // the rest of a3 (permute + pack)
    k_validate_pack_vmu<<<grid1d(c, n, 256), 256, 0, c->stream2>>>(vd, md, ud, n, vmc, verr);
    k_gather_vmu<<<grid1d(c, n, 256), 256, 0, c->stream2>>>(Bget<uint32_t>(c, B_PERM), n, vmc, ud, vm, uc);
    CUDA_TRY(cudaGetLastError());
    c->launches += 2;
  }
  CUDA_TRY(cudaEventRecord(c->ev_side[5], c->stream2));
  unsigned long long hc[C_NCOUNTERS];

  uint8_t* state = Bget<uint8_t>(c, B_STATE);
  if (c->state >= 2) {   // a repeated call: iterate again from the current h (lists stay valid)
    LAUNCH(k_init_iter, grid1d(c, n, 256), 256, 0, Bget<uint8_t>(c, B_TGT), n, Bget<float4>(c, B_XH),
           1.0f, h_cap(c), state, (float*)nullptr, Bget<float>(c, B_HLO), Bget<float>(c, B_HHI));
  }
  // a8: the h iteration, per particle on its neighbour list; re-walk particles whose root
  // lies beyond their list, until every particle has converged
  const float margin = solve_margin(c);
  int rounds = 0;
  long long unconv = 0, itmax = 0;
  CUDA_TRY(cudaEventRecord(c->ev[6], c->stream));
  if (c->state >= 2) {
    // a repeated call: the lists are recorded; solve on them from the current h
    hctr_zero(c);
    PhaseTimer _p(c, 1);
    LAUNCH(k_hsolve, gridfull((int64_t)c->n_groups * 32, HSOLVE_WARPS * 32), HSOLVE_WARPS * 32, 0,
           Bget<int4>(c, B_GROUPS), c->n_groups, Bget<float4>(c, B_XH), Bget<float>(c, B_HB), Bget<float>(c, B_HLO),
           Bget<float>(c, B_HHI), state, Bget<float>(c, B_NBR2), Bget<int>(c, B_NBCNT), c->nb_k,
           Bget<int64_t>(c, B_NBOFF), Bget<float>(c, B_NBOVF), c->cfg.n_ngb, c->cfg.n_ngb_tol, margin, h_cap(c),
           c->cfg.max_h_iter, Bget<unsigned long long>(c, B_HCTR));
    c->rg_valid = false;   // its re-walk particles are not in the group list
    if (c->n_ovfidx > 0)
      LAUNCH(k_hsolve_pool, gridfull((int64_t)c->n_ovfidx * 32, HSOLVE_WARPS * 32), HSOLVE_WARPS * 32, 0,
             Bget<int32_t>(c, B_OVFIDX), (int)c->n_ovfidx, Bget<float4>(c, B_XH), Bget<float>(c, B_HB),
             Bget<float>(c, B_HLO), Bget<float>(c, B_HHI), state, Bget<int>(c, B_NBCNT), Bget<int64_t>(c, B_NBOFF),
             Bget<float>(c, B_NBOVF), c->cfg.n_ngb, c->cfg.n_ngb_tol, margin, h_cap(c), c->cfg.max_h_iter,
             Bget<unsigned long long>(c, B_HCTR));
      c->rg_valid = false;   // its re-walk particles are not in the group list
  }
  // The first solve ran fused into the build's walk (lists.cuh); each round reads its
  // counters (one host round trip), records the lists of the particles whose root lies
  // beyond their list (a fused re-walk + solve) and the pool lists of repeat overflows.
  while (true) {
    unsigned long long hh[HC_N];
    read_dev(c, hh, Bget<unsigned long long>(c, B_HCTR), sizeof(hh));
    ++rounds;
    unconv += (long long)hh[HC_UNCONV];   // disjoint per round: an unconverged particle is never re-walked
    itmax = std::max(itmax, (long long)hh[HC_ITMAX]);
    c->h_evals = (int64_t)hh[HC_EVALS];   // cumulative over the build's walk and every round
    DBG("h solve round %d: unconverged %llu, re-walk %llu, pool %llu, max iterations %llu\n", rounds,
        hh[HC_UNCONV], hh[HC_REGROW], hh[HC_OVF], hh[HC_ITMAX]);
    if (hh[HC_REGROW] == 0 && hh[HC_OVF] == 0) break;
    if (rounds >= c->cfg.max_h_iter) {
      unconv += (long long)(hh[HC_REGROW] + hh[HC_OVF]);
      break;
    }
    hctr_reset(c);
    if (hh[HC_OVF] > 0) {
      nb_pool(c);
      PhaseTimer _p(c, 1);
      LAUNCH(k_hsolve_pool, gridfull((int64_t)c->n_ovfidx * 32, HSOLVE_WARPS * 32), HSOLVE_WARPS * 32, 0,
             Bget<int32_t>(c, B_OVFIDX), (int)c->n_ovfidx, Bget<float4>(c, B_XH), Bget<float>(c, B_HB),
             Bget<float>(c, B_HLO), Bget<float>(c, B_HHI), state, Bget<int>(c, B_NBCNT), Bget<int64_t>(c, B_NBOFF),
             Bget<float>(c, B_NBOVF), c->cfg.n_ngb, c->cfg.n_ngb_tol, margin, h_cap(c), c->cfg.max_h_iter,
             Bget<unsigned long long>(c, B_HCTR));
      c->rg_valid = false;   // its re-walk particles are not in the group list
    }
    if (hh[HC_REGROW] > 0) {
      nb_walk(c, HS_REGROW, (int64_t)hh[HC_REGROW]);
      c->list_rebuilds += (int64_t)hh[HC_REGROW];
    }
  }
  CUDA_TRY(cudaEventRecord(c->ev[7], c->stream));
  // a7 (first half): the interaction lists need only x and the final h (reach max(h_i, h_j)
  // with the owned particles' h; these are the force lists too when there is no halo), so
  // they are built while the side stream still copies v, m, u from the host
  float* hr = Bget<float>(c, B_HRCH);
  LAUNCH(k_reach_owned, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, c->n_own, Bget<float4>(c, B_XH),
         hr);
  build_union(c, hr);
  c->force_lists = c->n == c->n_own;
  // h is final: a pinned host h_out is copied back on the side stream during the density
  // loop (the ghost then skips h; a pageable copy would block the host)
  const bool h_early = is_pinned_host_ptr(h_out);
  if (h_early) {
    float* hs = B<float>(c, B_OUT0, c->n_own);
    LAUNCH(k_scatter_h_own, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, c->n_own, Bget<float4>(c, B_XH),
           hs);
    CUDA_TRY(cudaEventRecord(c->ev_side[2], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream2, c->ev_side[2], 0));
    CUDA_TRY(cudaMemcpyAsync(h_out, hs, c->n_own * sizeof(float), cudaMemcpyDeviceToHost, c->stream2));
    CUDA_TRY(cudaEventRecord(c->ev_side[3], c->stream2));
  }
  // join the side stream's v, m, u (checked, in cell order); their error bits are read with
  // the density kernel's counters below (one host round trip)
  CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_side[5], 0));
  (void)side;
  ctr_reset(c);
  // a9 ghost fused into the density kernel: the caller-order outputs and the force state
  std::vector<OutMap> maps;
  GhostOut go;
  const int64_t no = c->n_own;
  go.h = h_early ? nullptr : dev_out(c, h_out, no, B_OUT0, maps);
  go.rho = dev_out(c, rho_out, no, B_OUT1, maps);
  go.omega = dev_out(c, omega_out, no, B_OUT2, maps);
  go.nnbr = dev_out(c, n_nbr_out, no, B_OUT3, maps);
  go.div = dev_out(c, div_out, no, B_OUT4, maps);
  go.curl = dev_out(c, curl_out, 3 * no, B_OUT5, maps);
  go.perm = Bget<uint32_t>(c, B_PERM);
  go.n_own = no;
  go.h_o = B<float>(c, B_HFIN_O, n);
  go.g_o = B<float4>(c, B_GST_O, n);
  // the targets' force inputs in cell order straight from the epilogue; sph_force gathers
  // only when other particles (halo, inactive) need theirs
  go.xh = Bget<float4>(c, B_XH);
  go.fx = B<float4>(c, B_FX, n);
  go.fs = B<float4>(c, B_FS, n);
  go.hr = Bget<float>(c, B_HRCH);
  DensOut dout;
  memset(&dout, 0, sizeof(dout));
  dout.g = go;
  dout.u = uc;
  dout.gamma = c->cfg.gamma;
  dout.beps = c->cfg.balsara_eps;
  dout.n_t = (float)c->cfg.n_ngb;
  // N(h) re-check: twice the iteration's tolerance plus a few fp32 ulps of h (the bracket
  // stop at fp32 resolution) in N = n_t (h/h)^3
  dout.tol_check = 2.f * (float)c->cfg.n_ngb_tol + 24.f * (float)c->cfg.n_ngb * 1.1920929e-7f;
  CUDA_TRY(cudaEventRecord(c->ev[8], c->stream));
  {
    DbgTimer _t(c, "density kernel");
    const GroupLists G = group_lists(c);
    const bool diag = (c->cfg.flags & SPH_F_DIAGNOSTICS) != 0;
    auto kd = diag ? k_density<false, true> : k_density<false, false>;
    LAUNCH(kd, gridfull(G.ngroups, DENS_WARPS), DENS_WARPS * 32, 0, G, Bget<float4>(c, B_XH), vm,
           Bget<uint32_t>(c, B_PERM), Bget<uint8_t>(c, B_TGT), box3(c), dout, ctr(c));
  }
  CUDA_TRY(cudaEventRecord(c->ev[9], c->stream));
  if (c->defer_out) {
    // sph_step: the host copies run on the side stream behind the density kernel while the
    // force loop runs (its staging buffers are others); sph_step joins them at its end
    CUDA_TRY(cudaEventRecord(c->ev[3], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream2, c->ev[3], 0));
    for (auto& mp : maps)
      CUDA_TRY(cudaMemcpyAsync(mp.user, mp.dev, mp.bytes, cudaMemcpyDeviceToHost, c->stream2));
  } else {
    if (h_early) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_side[3], 0));   // the call ends after the h copy
    flush_out(c, maps, c->ev[3]);
    if (h_early) CUDA_TRY(cudaStreamSynchronize(c->stream2));
  }
  bool noconv = unconv > 0;
  CUDA_TRY(cudaMemcpyAsync(c->hpin, ctr(c), sizeof(unsigned long long) * C_NCOUNTERS, cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->hpin + C_NCOUNTERS, verr + C_ERR, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           c->stream));
  // the recorded neighbour-list entries in the same round trip
  CUDA_TRY(cudaMemcpyAsync(c->hpin + C_NCOUNTERS + 1, Bget<unsigned long long>(c, B_NBENT), sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  c->nb_entries = (int64_t)c->hpin[C_NCOUNTERS + 1];
  memcpy(hc, c->hpin, sizeof(hc));
  hc[C_ERR] |= c->hpin[C_NCOUNTERS];
  if ((hc[C_ERR] & (ERRBIT_NONFINITE | ERRBIT_MASS | ERRBIT_U)) && c->defer_out)
    cudaStreamSynchronize(c->stream2);   // no copy may outlive the failed call
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_NONFINITE), SPH_E_DOMAIN, "non-finite velocity");
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_MASS), SPH_E_DOMAIN, "mass <= 0 or non-finite");
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_U), SPH_E_DOMAIN, "internal energy <= 0 or non-finite");
  c->state = 2;
  const long long ndir = (long long)hc[C_NDIR];
  const long long cand = (long long)hc[C_CAND];
  const long long nbord_d = (long long)hc[C_BORDER_D], ncoinc = (long long)hc[C_COINC] / 2;
  const long long nbad = (long long)hc[C_UNCONV];
  if (nbad > 0 && !noconv) {   // an accepted step failed the N(h) re-check (R4): not converged
    noconv = true;
    unconv = nbad;
  }
  if (c->n > c->n_own && c->cfg.halo_width > 0.0) {
    // every owned particle's partners must be inside the received halo: the largest h of an
    // owned particle within h of a face must not exceed the halo width (k_hface)
    ctr_reset(c);
    LAUNCH(k_hface, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), Bget<float4>(c, B_XH), n, c->n_own,
           (float)c->cfg.slab_lo, (float)c->cfg.slab_hi, ctr(c));
    unsigned long long hh[C_NCOUNTERS];
    ctr_read(c, hh);
    c->h_own_max = as_float(hh[C_HMAXBITS]);
    SPH_REQUIRE(as_float(hh[C_HMAXBITS]) <= c->cfg.halo_width, SPH_E_NOCONV,
                "halo too narrow: an owned h = " + std::to_string(as_float(hh[C_HMAXBITS])) +
                    " within h of a slab face exceeds cfg.halo_width");
  }
  phase_resolve(c);
  if (st) {
    memset(st, 0, sizeof(*st));
    fill_struct_stats(c, st);
    st->ms_kernel_walk_nb = c->ms_phase[0];
    st->ms_kernel_hsolve = c->ms_phase[1];
    st->ms_kernel_walk_union = c->ms_phase[2];
    st->n_nb_entries = c->nb_entries;
    st->n_h_evals = c->h_evals;
    st->n_walk_launches = c->walk_launches;
    st->cells_reused = c->cells_reused ? 1 : 0;
    st->ms_kernel_sort = c->ms_phase[3];
    st->sort_key_bits = c->sort_bits;
    st->sort_passes = c->sort_passes;
    if (c->cfg.flags & SPH_F_COUNT_CANDIDATES) {
      unsigned long long wr[2];
      read_dev(c, wr, Bget<unsigned long long>(c, B_WALKRAW), sizeof(wr));
      st->n_nb_sources = (int64_t)wr[0];
      st->n_union_sources = (int64_t)wr[1];
    }
    st->n_directed = ndir;
    st->n_borderline = nbord_d;
    st->n_coincident = ncoinc;
    st->n_candidates = cand;
    st->n_candidates_density_full = cand;
    st->n_unconverged = noconv ? unconv : 0;
    st->h_iters = (int)itmax;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    st->ms_build = ms;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
    st->ms_density = ms;
    cudaEventElapsedTime(&ms, c->ev[8], c->ev[9]);
    st->ms_kernel_density_full = ms;
  }
  if (noconv) {
    c->err = "h iteration did not converge in max_h_iter iterations: " + std::to_string(unconv) + " particles";
    return SPH_E_NOCONV;
  }
  API_END
  return SPH_OK;
}

// Force inputs in cell order (halo particles carry the imported state); the interaction
// lists are rebuilt only when halo particles' h entered after the density loop.
static void prepare_force(sph_ctx* c) {
  const int64_t n = c->n;
  float4* fx = B<float4>(c, B_FX, n);
  float4* fs = B<float4>(c, B_FS, n);
  float* hr = Bget<float>(c, B_HRCH);
  // every particle a target: the density epilogue wrote them all
  if (c->n != c->n_own || c->has_active)
    LAUNCH(k_gather_force, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, Bget<float4>(c, B_XH),
           Bget<float>(c, B_HFIN_O), Bget<float4>(c, B_GST_O), fx, fs, hr);
  if (!c->force_lists) build_union(c, hr);
  c->force_lists = true;
}

int sph_force(sph_ctx* ctx, float* a_out, float* dudt_out, float* vsig_out, int32_t* n_nbr_force_out,
              sph_stats* st) {
  API_BEGIN(ctx)
  if (c->has_active) {
    const void* outs[4] = {a_out, dudt_out, vsig_out, n_nbr_force_out};
    for (const void* o : outs)
      SPH_REQUIRE(!o || is_device_ptr(o), SPH_E_ARG, "with an active mask the outputs must be device arrays");
  }
  SPH_REQUIRE(c->state >= 2, SPH_E_STATE, "sph_force before sph_density");
  SPH_REQUIRE(a_out && dudt_out, SPH_E_ARG, "required pointer is NULL");
  const int64_t no = c->n_own;
  CUDA_TRY(cudaEventRecord(c->ev[4], c->stream));
  DbgTimer _tf(c, "force call");
  if (c->state == 2) {
    prepare_force(c);
    c->state = 3;
  }
  std::vector<OutMap> maps;
  ForceOut fo;
  fo.a = dev_out(c, a_out, 3 * no, B_FOUT0, maps);
  fo.dudt = dev_out(c, dudt_out, no, B_FOUT1, maps);
  fo.vsig = dev_out(c, vsig_out, no, B_FOUT2, maps);
  fo.nnbr = dev_out(c, n_nbr_force_out, no, B_FOUT3, maps);
  fo.perm = Bget<uint32_t>(c, B_PERM);
  fo.n_own = no;
  fo.tgt = Bget<uint8_t>(c, B_TGT);
  ctr_reset(c);
  const GroupLists G = group_lists(c);
  CUDA_TRY(cudaEventRecord(c->ev[10], c->stream));
  {
    DbgTimer _t(c, "force kernel");
    if (c->cfg.flags & SPH_F_SYMMETRIC) {
      // every unordered pair once, both particles updated (interact.cuh k_force_sym)
      const int64_t n = c->n;
      ForceSym Y;
      Y.pgroup = B<int>(c, B_PGROUP, n);
      LAUNCH(k_pgroup, gridfull((int64_t)G.ngroups * 32, 256), 256, 0, G.groups, G.ngroups, B<int>(c, B_PGROUP, n));
      Y.ia = B<float4>(c, B_SYM_IA, n);
      Y.ivs = B<float>(c, B_SYM_IVS, n);
      Y.icnt = B<int>(c, B_SYM_ICNT, n);
      Y.ja = B<float4>(c, B_SYM_JA, n);
      Y.jvs = B<unsigned>(c, B_SYM_JVS, n);
      Y.jcnt = B<int>(c, B_SYM_JCNT, n);
      CUDA_TRY(cudaMemsetAsync(Y.ja, 0, n * sizeof(float4), c->stream));
      CUDA_TRY(cudaMemsetAsync(Y.jvs, 0, n * sizeof(unsigned), c->stream));
      CUDA_TRY(cudaMemsetAsync(Y.jcnt, 0, n * sizeof(int), c->stream));
      auto ks = (c->cfg.flags & SPH_F_DIAGNOSTICS) ? k_force_sym<true> : k_force_sym<false>;
      LAUNCH(ks, gridfull(G.ngroups, FORCE_WARPS), FORCE_WARPS * 32, 0, G, Bget<float4>(c, B_FX), Bget<float4>(c, B_VM),
             Bget<float4>(c, B_FS), c->cfg.alpha, box3(c), fo, Y, ctr(c));
      LAUNCH(k_force_sym_finish, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, Bget<uint8_t>(c, B_TGT), Y,
             fo);
    } else {
      auto kf = (c->cfg.flags & SPH_F_DIAGNOSTICS) ? k_force<true> : k_force<false>;
      LAUNCH(kf, gridfull(G.ngroups, FORCE_WARPS), FORCE_WARPS * 32, 0, G, Bget<float4>(c, B_FX),
             Bget<float4>(c, B_VM), Bget<float4>(c, B_FS), c->cfg.alpha, box3(c), fo, ctr(c));
    }
  }
  CUDA_TRY(cudaEventRecord(c->ev[11], c->stream));
  // the counters come back with the outputs' copies (one round trip)
  CUDA_TRY(cudaMemcpyAsync(c->hpin, ctr(c), sizeof(unsigned long long) * C_NCOUNTERS, cudaMemcpyDeviceToHost,
                           c->stream));
  flush_out(c, maps, c->ev[5]);
  if (maps.empty()) sync(c);
  unsigned long long hc[C_NCOUNTERS];
  memcpy(hc, c->hpin, sizeof(hc));
  SPH_REQUIRE(!(hc[C_ERR] & (1ull << 20)), SPH_E_CUDA, "interaction list count/fill mismatch");
  DBG("force: groups %d cand %llu pairs %llu; host syncs so far %lld, launches %lld\n", c->n_groups, hc[C_CAND],
      hc[C_NFORCE] / 2, (long long)g_syncs, (long long)c->launches);
  c->ms_phase[2] = 0.0;
  phase_resolve(c);
  if (st) {
    memset(st, 0, sizeof(*st));
    fill_struct_stats(c, st);
    st->ms_kernel_walk_union = c->ms_phase[2];
    st->n_pairs = (int64_t)(hc[C_NFORCE] / 2);
    st->n_candidates = (int64_t)hc[C_CAND];
    st->n_borderline_force = (int64_t)(hc[C_BORDER_F] / 2);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]);
    st->ms_force = ms;
    cudaEventElapsedTime(&ms, c->ev[10], c->ev[11]);
    st->ms_kernel_force = ms;
  }
  API_END
  return SPH_OK;
}

// One evaluation with the host <-> device copies overlapped (include/sph.h): v, m, u go up on
// the side stream while the cells and neighbour lists are built; the density's host outputs
// come down on the side stream while the force loop runs.
int sph_step(sph_ctx* ctx, int64_t n, const float* x, const float* h0, const float* v, const float* m,
             const float* u, float* h_out, float* rho_out, float* a_out, float* dudt_out, sph_stats* st_density,
             sph_stats* st_force) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n > 0 && x && v && m && u && h_out && rho_out && a_out && dudt_out, SPH_E_ARG,
              "required pointer is NULL");
  // v, m, u are staged by the build right after it enqueued x (copies queued before x would
  // delay the build: one copy engine serves both streams in order)
  c->pre_in[0] = v;
  c->pre_in[1] = m;
  c->pre_in[2] = u;
  c->pre_pending = true;
  c->pre_ready = false;
  API_END
  ctx->in_step = true;
  int rc = sph_build_cells(ctx, n, x, h0);
  ctx->in_step = false;
  ctx->pre_pending = false;
  if (rc != SPH_OK) {
    ctx->pre_ready = false;
    return rc;
  }
  ctx->defer_out = true;
  const int rd = sph_density(ctx, v, m, u, h_out, rho_out, nullptr, nullptr, nullptr, nullptr, st_density);
  ctx->defer_out = false;
  if (rd != SPH_OK && rd != SPH_E_NOCONV) {
    cudaStreamSynchronize(ctx->stream2);
    return rd;
  }
  const int rf = sph_force(ctx, a_out, dudt_out, nullptr, nullptr, st_force);
  if (cudaStreamSynchronize(ctx->stream2) != cudaSuccess && rf == SPH_OK) {   // the density's host outputs
    ctx->err = std::string("sph_step: ") + cudaGetErrorString(cudaGetLastError());
    return SPH_E_CUDA;
  }
  return rf != SPH_OK ? rf : rd;
}

int sph_guess_h(sph_ctx* ctx, int64_t n, const float* x, float* h_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n > 0 && x && h_out, SPH_E_ARG, "bad argument");
  SPH_REQUIRE(n <= (1ll << SPH_IDX_BITS), SPH_E_ARG, "n > 2^27 particles in one context");
  c->n = n;
  c->n_own = n;
  c->state = 0;
  float h0max = 0.f;
  load_inputs(c, x, nullptr, &h0max);
  sort_particles(c, 0.f, false);
  build_nodes(c, false);
  LAUNCH(k_guess_h, gridfull((int64_t)c->n_nodes * 32, 256), 256, 0, c->n_nodes, nodes(c), level_geom(c),
         c->cfg.n_ngb, (int)c->cfg.n_ngb, h_cap(c), Bget<float4>(c, B_XH));
  std::vector<OutMap> maps;
  float* o = dev_out(c, h_out, n, B_OUT0, maps);
  LAUNCH(k_scatter_h, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, Bget<float4>(c, B_XH), o);
  flush_out(c, maps, c->ev[10]);
  sync(c);
  API_END
  return SPH_OK;
}

// the two face selections of sph_halo_select (width > 0) and sph_slab_leavers (width == 0)
static void face_select(sph_ctx* c, int64_t n, const float* x, double lo, double hi, double width,
                        int32_t* idx_lo_out, int32_t* idx_hi_out, int64_t* counts_out);

int sph_halo_select(sph_ctx* ctx, int64_t n, const float* x, double lo, double hi, double width,
                    int32_t* idx_lo_out, int32_t* idx_hi_out, int64_t* counts_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n > 0 && x && idx_lo_out && idx_hi_out && counts_out, SPH_E_ARG, "bad argument");
  SPH_REQUIRE(hi > lo && width > 0.0, SPH_E_ARG, "need hi > lo and width > 0");
  face_select(c, n, x, lo, hi, width, idx_lo_out, idx_hi_out, counts_out);
  API_END
  return SPH_OK;
}

int sph_slab_leavers(sph_ctx* ctx, int64_t n, const float* x, double lo, double hi, int32_t* idx_lo_out,
                     int32_t* idx_hi_out, int64_t* counts_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && idx_lo_out && idx_hi_out && counts_out && (n == 0 || x), SPH_E_ARG, "bad argument");
  SPH_REQUIRE(hi > lo, SPH_E_ARG, "need hi > lo");
  if (n == 0) {
    counts_out[0] = counts_out[1] = 0;
    return SPH_OK;
  }
  face_select(c, n, x, lo, hi, 0.0, idx_lo_out, idx_hi_out, counts_out);
  API_END
  return SPH_OK;
}

// ------------------------------------------------------------------ CUDA IPC (peer stores) -----
int sph_ipc_alloc(sph_ctx* ctx, int64_t bytes, void** dev_ptr, uint8_t* handle) {
  API_BEGIN(ctx)
  SPH_REQUIRE(bytes > 0 && dev_ptr && handle, SPH_E_ARG, "bad argument");
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, (size_t)bytes));   // its own allocation: the handle names exactly it
  c->ipc_own.push_back(p);
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, p));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *dev_ptr = p;
  API_END
  return SPH_OK;
}

int sph_ipc_open(sph_ctx* ctx, const uint8_t* handle, void** dev_ptr) {
  API_BEGIN(ctx)
  SPH_REQUIRE(handle && dev_ptr, SPH_E_ARG, "bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->ipc_open.push_back(p);
  *dev_ptr = p;
  API_END
  return SPH_OK;
}

int sph_ipc_event_create(sph_ctx* ctx, int32_t* id, uint8_t* handle) {
  API_BEGIN(ctx)
  SPH_REQUIRE(id && handle, SPH_E_ARG, "bad argument");
  cudaEvent_t e;
  CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess));
  c->ipc_ev.push_back(e);
  cudaIpcEventHandle_t h;
  CUDA_TRY(cudaIpcGetEventHandle(&h, e));
  static_assert(sizeof(h) == 64, "IPC event handle size");
  memcpy(handle, &h, sizeof(h));
  *id = (int32_t)c->ipc_ev.size() - 1;
  API_END
  return SPH_OK;
}

int sph_ipc_event_open(sph_ctx* ctx, const uint8_t* handle, int32_t* id) {
  API_BEGIN(ctx)
  SPH_REQUIRE(id && handle, SPH_E_ARG, "bad argument");
  cudaIpcEventHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaEvent_t e;
  CUDA_TRY(cudaIpcOpenEventHandle(&e, h));
  c->ipc_ev.push_back(e);
  *id = (int32_t)c->ipc_ev.size() - 1;
  API_END
  return SPH_OK;
}

int sph_ipc_event_record(sph_ctx* ctx, int32_t id) {
  API_BEGIN(ctx)
  SPH_REQUIRE(id >= 0 && id < (int32_t)c->ipc_ev.size(), SPH_E_ARG, "unknown event");
  CUDA_TRY(cudaEventRecord(c->ipc_ev[id], c->stream));
  API_END
  return SPH_OK;
}

int sph_ipc_event_wait(sph_ctx* ctx, int32_t id) {
  API_BEGIN(ctx)
  SPH_REQUIRE(id >= 0 && id < (int32_t)c->ipc_ev.size(), SPH_E_ARG, "unknown event");
  CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ipc_ev[id], 0));
  API_END
  return SPH_OK;
}

int sph_halo_required(sph_ctx* ctx, double* h_max) {
  API_BEGIN(ctx)
  SPH_REQUIRE(h_max, SPH_E_ARG, "h_max is NULL");
  *h_max = c->h_own_max;
  API_END
  return SPH_OK;
}

int sph_set_halo_width(sph_ctx* ctx, double width) {
  API_BEGIN(ctx)
  SPH_REQUIRE(width >= 0.0 && std::isfinite(width), SPH_E_ARG, "width must be finite and >= 0");
  c->cfg.halo_width = width;
  API_END
  return SPH_OK;
}

int sph_x_histogram_weighted(sph_ctx* ctx, int64_t n, const float* x, const int32_t* w, double lo, double hi,
                             int32_t nbins, int64_t* hist_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && nbins > 0 && hist_out && (n == 0 || (x && w)) && hi > lo, SPH_E_ARG, "bad argument");
  unsigned long long* hd = B<unsigned long long>(c, B_TMPL1, nbins);
  CUDA_TRY(cudaMemsetAsync(hd, 0, nbins * sizeof(unsigned long long), c->stream));
  if (n > 0) {
    const float* xd = dev_in(c, x, 3 * n, B_XIN);
    const int32_t* wd = dev_in(c, w, n, B_WIN);
    LAUNCH(k_x_hist_w, grid1d(c, n, 256), 256, 0, xd, wd, n, (float)lo, (float)hi, nbins, hd);
  }
  std::vector<OutMap> maps;
  int64_t* o = dev_out(c, hist_out, nbins, B_OUT3, maps);
  CUDA_TRY(cudaMemcpyAsync(o, hd, nbins * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream));
  flush_out(c, maps, c->ev[10]);
  sync(c);
  API_END
  return SPH_OK;
}

}  // extern "C"

static void face_select(sph_ctx* c, int64_t n, const float* x, double lo, double hi, double width,
                        int32_t* idx_lo_out, int32_t* idx_hi_out, int64_t* counts_out) {
  const float* xd = dev_in(c, x, 3 * n, B_XIN);
  int* flo = B<int>(c, B_TMPI0, n);
  int* fhi = B<int>(c, B_TMPI1, n);
  int* slo = B<int>(c, B_GFLAG, n);
  int* shi = B<int>(c, B_GSEL, n);
  LAUNCH(k_halo_flags, grid1d(c, n, 256), 256, 0, xd, n, (float)lo, (float)hi, (float)width, flo, fhi);
  const int nlo = scan_excl<int>(c, flo, slo, n);
  const int nhi = scan_excl<int>(c, fhi, shi, n);
  std::vector<OutMap> maps;
  int32_t* olo = dev_out(c, idx_lo_out, std::max(nlo, 1), B_OUT0, maps);
  int32_t* ohi = dev_out(c, idx_hi_out, std::max(nhi, 1), B_OUT1, maps);
  for (auto& mp : maps) mp.bytes = (mp.user == (void*)idx_lo_out ? (size_t)nlo : (size_t)nhi) * sizeof(int32_t);
  LAUNCH(k_compact_idx, grid1d(c, n, 256), 256, 0, flo, slo, n, olo);
  LAUNCH(k_compact_idx, grid1d(c, n, 256), 256, 0, fhi, shi, n, ohi);
  flush_out(c, maps, c->ev[10]);
  sync(c);
  counts_out[0] = nlo;
  counts_out[1] = nhi;
}

extern "C" {

int sph_halo_pack(sph_ctx* ctx, const float* x, const float* v, const float* m, const float* u, const float* h0,
                  int64_t k, const int32_t* idx, float* out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(k >= 0, SPH_E_ARG, "k < 0");
  if (k == 0) return SPH_OK;
  SPH_REQUIRE(x && v && m && u && idx && out, SPH_E_ARG, "required pointer is NULL");
  const void* ptrs[7] = {x, v, m, u, idx, out, h0};
  for (int i = 0; i < 7; ++i)
    SPH_REQUIRE(!ptrs[i] || is_device_ptr(ptrs[i]), SPH_E_ARG, "sph_halo_pack: arrays must be device memory");
  LAUNCH(k_halo_pack, grid1d(c, k, 256), 256, 0, x, v, m, u, h0, idx, k, out);
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

int sph_export_state(sph_ctx* ctx, int64_t k, const int32_t* idx, float* state_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->state >= 2, SPH_E_STATE, "sph_export_state before sph_density");
  SPH_REQUIRE(k >= 0 && (k == 0 || (idx && state_out)), SPH_E_ARG, "bad argument");
  if (k == 0) return SPH_OK;
  const int32_t* id = dev_in(c, idx, k, B_TMPI0);
  std::vector<OutMap> maps;
  float* o = dev_out(c, state_out, 5 * k, B_OUT2, maps);
  LAUNCH(k_export_state, grid1d(c, k, 256), 256, 0, id, k, Bget<float>(c, B_HFIN_O), Bget<float4>(c, B_GST_O), o);
  flush_out(c, maps, c->ev[10]);
  sync(c);
  API_END
  return SPH_OK;
}

int sph_import_halo_state(sph_ctx* ctx, const float* state) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->state >= 2, SPH_E_STATE, "sph_import_halo_state before sph_density");
  const int64_t k = c->n - c->n_own;
  if (k == 0) return SPH_OK;
  SPH_REQUIRE(state != nullptr, SPH_E_ARG, "state == NULL");
  const float* sd = dev_in(c, state, 5 * k, B_TMPL0);
  LAUNCH(k_import_state, grid1d(c, k, 256), 256, 0, sd, k, c->n_own, Bget<float>(c, B_HFIN_O),
         Bget<float4>(c, B_GST_O));
  c->force_lists = false;
  if (c->state > 2) c->state = 2;   // force inputs must be gathered again
  sync(c);
  API_END
  return SPH_OK;
}

int sph_x_histogram(sph_ctx* ctx, int64_t n, const float* x, double lo, double hi, int32_t nbins,
                    int64_t* hist_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && nbins > 0 && hist_out && (n == 0 || x) && hi > lo, SPH_E_ARG, "bad argument");
  unsigned long long* hd = B<unsigned long long>(c, B_TMPL1, nbins);
  CUDA_TRY(cudaMemsetAsync(hd, 0, nbins * sizeof(unsigned long long), c->stream));
  if (n > 0) {
    const float* xd = dev_in(c, x, 3 * n, B_XIN);
    LAUNCH(k_x_hist, grid1d(c, n, 256), 256, 0, xd, n, (float)lo, (float)hi, nbins, hd);
  }
  std::vector<OutMap> maps;
  int64_t* o = dev_out(c, hist_out, nbins, B_OUT3, maps);
  CUDA_TRY(cudaMemcpyAsync(o, hd, nbins * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream));
  flush_out(c, maps, c->ev[10]);
  sync(c);
  API_END
  return SPH_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ pseudo-Verlet -------
// sph_update_cells: new positions (and h) of the same particles; when no particle moved by
// more than a tenth of the smallest h since the last full build, the sort, hierarchy and
// groups are kept and every node test is widened by that drift; else a full
// build. Then the neighbour lists and h iteration as in sph_build_cells.
int sph_update_cells(sph_ctx* ctx, const float* x, const float* h0) {
  API_BEGIN(ctx)
  SPH_REQUIRE(x && h0, SPH_E_ARG, "x or h0 NULL");
  SPH_REQUIRE(!c->has_active || c->n_active_for == c->n_own, SPH_E_ARG,
              "an active mask (sph_set_active) must cover the n_own particles of the last build");
  const bool can = c->state >= 1 && c->n == c->n_own && c->n_sorted == 0;
  if (!can) {
    c->cells_reused = false;
    return sph_build_cells_halo(ctx, c->n_own, 0, x, h0);
  }
  const int64_t n = c->n;
  float h0max = 0.f;
  const bool need_guess = load_inputs(c, x, h0, &h0max, true);
  SPH_REQUIRE(!need_guess, SPH_E_ARG, "sph_update_cells needs every h0 > 0");
  unsigned long long hc[C_NCOUNTERS];
  ctr_reset(c);
  LAUNCH(k_hrange, grid1d(c, n, 256), 256, 0, c->hin, n, ctr(c));
  ctr_read(c, hc);
  const float hmin = as_float(hc[C_HMINBITS]);
  if (!c->xref_valid) {   // the build's positions (xh holds them until the first update)
    CUDA_TRY(cudaMemcpyAsync(B<float4>(c, B_XREF, n), Bget<float4>(c, B_XH), n * sizeof(float4),
                             cudaMemcpyDeviceToDevice, c->stream));
    c->xref_valid = true;
  }
  ctr_reset(c);
  LAUNCH(k_update_pos, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, c->xin, c->hin,
         Bget<float4>(c, B_XREF), (float)c->cfg.box[0], (float)c->cfg.box[1],
         (float)c->cfg.box[2], Bget<float4>(c, B_XH), ctr(c));
  ctr_read(c, hc);
  const float drift = as_float(hc[C_HMAXBITS]);
  if (!(drift <= 0.1f * hmin)) {
    c->cells_reused = false;
    return sph_build_cells_halo(ctx, c->n_own, 0, x, h0);
  }
  c->cells_reused = true;
  c->skin = 1.7320508f * drift * 1.0001f;   // |d| <= sqrt(3) max component
  c->state = 0;
  c->force_lists = false;
  c->pool = 0;
  c->list_rebuilds = 0;
  CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
  phase_reset(c);
  CUDA_TRY(cudaMemsetAsync(B<unsigned long long>(c, B_NBENT, 1), 0, sizeof(unsigned long long), c->stream));
  {
    float* hb = B<float>(c, B_HB, n);
    CUDA_TRY(cudaMemsetAsync(B<int64_t>(c, B_NBOFF, n), 0xff, n * sizeof(int64_t), c->stream));
    CUDA_TRY(cudaMemsetAsync(B<uint8_t>(c, B_SHRUNK, n), 0, n, c->stream));
    CUDA_TRY(cudaMemsetAsync(B<int64_t>(c, B_OVFC, n), 0, n * sizeof(int64_t), c->stream));
    c->ovf_used = 0;
    c->n_ovfidx = 0;
    LAUNCH(k_make_tgt, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, c->n_own,
           c->has_active ? Bget<uint8_t>(c, B_ACTIVE) : (const uint8_t*)nullptr, B<uint8_t>(c, B_TGT, n));
    LAUNCH(k_init_iter, grid1d(c, n, 256), 256, 0, Bget<uint8_t>(c, B_TGT), n, Bget<float4>(c, B_XH),
           c->cfg.h_margin, h_cap(c), Bget<uint8_t>(c, B_STATE), hb, Bget<float>(c, B_HLO), Bget<float>(c, B_HHI));
  }
  hctr_zero(c);
  CUDA_TRY(cudaMemsetAsync(B<unsigned long long>(c, B_WALKRAW, 2), 0, 2 * sizeof(unsigned long long), c->stream));
  nb_walk(c, -1);
  c->state = 1;
  CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
  sync(c);
  API_END
  return SPH_OK;
}

// ------------------------------------------------------------------ introspection -----
int sph_debug_export(sph_ctx* ctx, int32_t what, void* out, int64_t cap, int64_t* count) {
  API_BEGIN(ctx)
  SPH_REQUIRE(count != nullptr, SPH_E_ARG, "count == NULL");
  SPH_REQUIRE(c->state >= 1, SPH_E_STATE, "sph_debug_export before sph_build_cells");
  int id = -1;
  int64_t cnt = 0;
  size_t esz = 0;
  switch (what) {
    case SPH_X_PERM: id = B_PERM; cnt = c->n; esz = 4; break;
    case SPH_X_GROUPS: id = B_GROUPS; cnt = c->n_groups; esz = 16; break;
    case SPH_X_LIST_OFF: id = B_GOFF; cnt = c->state >= 2 ? c->n_groups : 0; esz = 8; break;
    case SPH_X_LIST_LEN: id = B_GLEN; cnt = c->state >= 2 ? c->n_groups : 0; esz = 4; break;
    case SPH_X_LIST: id = B_LIST; cnt = c->state >= 2 ? c->pool : 0; esz = 4; break;
    case SPH_X_NODES: id = B_N_REC; cnt = c->n_nodes; esz = 16; break;
    case SPH_X_SORTOFF: id = B_N_SORTOFF; cnt = c->n_nodes; esz = 8; break;
    case SPH_X_SORTED: id = B_SORTED; cnt = c->n_sorted; esz = sizeof(SortEntry); break;
    case SPH_X_XH: id = B_XH; cnt = c->n; esz = 16; break;
    default: SPH_REQUIRE(false, SPH_E_ARG, "unknown sph_debug_export item");
  }
  *count = cnt;
  if (cnt > 0 && cap >= cnt) {
    SPH_REQUIRE(out != nullptr, SPH_E_ARG, "out == NULL");
    CUDA_TRY(cudaMemcpyAsync(out, c->b[id].p, (size_t)cnt * esz, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  }
  API_END
  return SPH_OK;
}

// ------------------------------------------------------------------ f2 ablation ----------
int sph_pair_ablation(sph_ctx* ctx, int32_t sorted, float* rho_out, int64_t* counts_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->state >= 2, SPH_E_STATE, "sph_pair_ablation before sph_density");
  SPH_REQUIRE(counts_out && (sorted == 0 || sorted == 1), SPH_E_ARG, "bad argument");
  const int64_t n = c->n;
  // grid edge >= the largest h, with a relative slack for the fp32 binning (R19)
  ctr_reset(c);
  LAUNCH(k_hrange, grid1d(c, n, 256), 256, 0, Bget<float>(c, B_HRCH), n, ctr(c));
  unsigned long long hc[C_NCOUNTERS];
  ctr_read(c, hc);
  const double hmax = (double)as_float(hc[C_HMAXBITS]) * (1.0 + 1e-5);
  int nc[3];
  for (int k = 0; k < 3; ++k) nc[k] = std::max(3, (int)floor(c->cfg.box[k] / hmax));
  const int ncell = nc[0] * nc[1] * nc[2];
  int* cell = B<int>(c, B_TMPI0, n);
  int* ccount = B<int>(c, B_GFLAG, ncell);
  int* cstart = B<int>(c, B_GSEL, ncell);
  int* cfill = B<int>(c, B_RGL, std::max<int64_t>(ncell, 2 * (int64_t)std::max(c->n_groups, 1)));
  int* order = B<int>(c, B_TMPI1, n);
  CUDA_TRY(cudaMemsetAsync(ccount, 0, ncell * sizeof(int), c->stream));
  const float4* xh = Bget<float4>(c, B_XH);
  LAUNCH(k_ab_cells, grid1d(c, n, 256), 256, 0, xh, n, nc[0], nc[1], nc[2], (float)(nc[0] / c->cfg.box[0]),
         (float)(nc[1] / c->cfg.box[1]), (float)(nc[2] / c->cfg.box[2]), cell, ccount);
  scan_excl<int>(c, ccount, cstart, ncell);
  CUDA_TRY(cudaMemsetAsync(cfill, 0, ncell * sizeof(int), c->stream));
  LAUNCH(k_ab_scatter, grid1d(c, n, 256), 256, 0, cell, n, cstart, cfill, order);
  AbParams P;
  memset(&P, 0, sizeof(P));
  P.nx = nc[0];
  P.ny = nc[1];
  P.nz = nc[2];
  for (int k = 0; k < 3; ++k) P.L[k] = (float)c->cfg.box[k];
  P.cstart = cstart;
  P.ccount = ccount;
  P.xh = xh;
  P.vm = Bget<float4>(c, B_VM);
  P.order = order;
  P.mode = sorted;
  float presort_ms = 0.f;
  if (sorted) {
    // the 13 presorted directions of every cell: one radix sort per direction of
    // (cell, projection) keys
    uint32_t* ls = B<uint32_t>(c, B_ABLIST, (size_t)13 * n * 2);   // [13][n] lists then [13][n] projections
    float* lp = reinterpret_cast<float*>(ls + (size_t)13 * n);
    int cbits = 0;
    while ((1 << cbits) < ncell) ++cbits;
    CUDA_TRY(cudaEventRecord(c->ev[10], c->stream));
    for (int d = 0; d < 13; ++d) {
      uint64_t* k0 = B<uint64_t>(c, B_KEYS0, n);
      uint64_t* k1 = B<uint64_t>(c, B_KEYS1, n);
      uint32_t* v0 = B<uint32_t>(c, B_VALS0, n);
      uint32_t* v1 = B<uint32_t>(c, B_VALS1, n);
      LAUNCH(k_ab_keys, grid1d(c, n, 256), 256, 0, xh, order, n, cell, nc[0], nc[1], (float)(c->cfg.box[0] / nc[0]),
             (float)(c->cfg.box[1] / nc[1]), (float)(c->cfg.box[2] / nc[2]), d, k0, v0);
      radix_sort(c, k0, v0, k1, v1, n, 32 + cbits);
      LAUNCH(k_ab_unpack, grid1d(c, n, 256), 256, 0, k0, v0, n, ls + (size_t)d * n, lp + (size_t)d * n);
    }
    CUDA_TRY(cudaEventRecord(c->ev[11], c->stream));
    sync(c);
    cudaEventElapsedTime(&presort_ms, c->ev[10], c->ev[11]);
    P.sorted = ls;
    P.proj = lp;
  }
  float* rs = B<float>(c, B_OUT4, n);
  CUDA_TRY(cudaMemsetAsync(rs, 0, n * sizeof(float), c->stream));
  P.rho_sum = rs;
  unsigned long long* ac = B<unsigned long long>(c, B_TMPL0, 16);
  CUDA_TRY(cudaMemsetAsync(ac, 0, 16 * sizeof(unsigned long long), c->stream));
  P.ctr = ac;
  CUDA_TRY(cudaEventRecord(c->ev[10], c->stream));
  LAUNCH(k_ab_pairs, gridfull((int64_t)ncell * 14 * 32, 256), 256, 0, P, ncell);
  CUDA_TRY(cudaEventRecord(c->ev[11], c->stream));
  std::vector<OutMap> maps;
  if (rho_out) {
    float* ro = dev_out(c, rho_out, c->n_own, B_OUT5, maps);
    LAUNCH(k_ab_finish, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, c->n_own, xh, P.vm, rs, ro);
  }
  flush_out(c, maps, c->ev[5]);
  unsigned long long h[16];
  CUDA_TRY(cudaMemcpyAsync(h, ac, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev[10], c->ev[11]);
  for (int k = 0; k < AB_N; ++k) counts_out[k] = (int64_t)h[k];
  counts_out[11] = nc[0];
  counts_out[12] = (int64_t)(ms * 1e6);
  counts_out[13] = (int64_t)(presort_ms * 1e6);
  counts_out[14] = counts_out[15] = 0;
  API_END
  return SPH_OK;
}

// ------------------------------------------------------------------ time-step limiter --
int sph_neighbour_min(sph_ctx* ctx, const float* val, float* out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->state >= 3, SPH_E_STATE, "sph_neighbour_min before sph_force");
  SPH_REQUIRE(val && out && is_device_ptr(val) && is_device_ptr(out), SPH_E_ARG,
              "sph_neighbour_min: val and out must be device arrays");
  const GroupLists G = group_lists(c);
  LAUNCH(k_scatter_min, gridfull(G.ngroups, 8), 256, 0, G, Bget<float4>(c, B_FX), Bget<uint32_t>(c, B_PERM),
         Bget<uint8_t>(c, B_TGT), val, box3(c), reinterpret_cast<unsigned*>(out));
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

// ------------------------------------------------------------------ active subset -----
int sph_set_active(sph_ctx* ctx, int64_t n, const uint8_t* active) {
  API_BEGIN(ctx)
  if (!active) {
    c->has_active = false;
    c->n_active_for = 0;
    return SPH_OK;
  }
  SPH_REQUIRE(n > 0, SPH_E_ARG, "n <= 0");
  uint8_t* d = B<uint8_t>(c, B_ACTIVE, n);
  CUDA_TRY(cudaMemcpyAsync(d, active, n, cudaMemcpyDefault, c->stream));
  sync(c);
  c->has_active = true;
  c->n_active_for = n;
  API_END
  return SPH_OK;
}

// ------------------------------------------------------------------ time step ---------
// SURVEY 8(f) f1 (first part): velocity-Verlet kick / drift and the Eq. 6 time step on the
// caller's device arrays; the density and force calls in between are the hot path.

int sph_kick(sph_ctx* ctx, int64_t n, float* v, float* u, const float* a, const float* dudt, float dt) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && (n == 0 || (v && a)) && (!u || dudt), SPH_E_ARG, "bad argument");
  SPH_REQUIRE(n == 0 || (is_device_ptr(v) && is_device_ptr(a) && (!u || (is_device_ptr(u) && is_device_ptr(dudt)))),
              SPH_E_ARG, "sph_kick: arrays must be device memory");
  if (n > 0) LAUNCH(k_kick, grid1d(c, n, 256), 256, 0, n, v, u, a, dudt, dt);
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

int sph_kick_each(sph_ctx* ctx, int64_t n, float* v, float* u, const float* a, const float* dudt, const float* dt) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && (n == 0 || (v && a && dt)) && (!u || dudt), SPH_E_ARG, "bad argument");
  SPH_REQUIRE(n == 0 || (is_device_ptr(v) && is_device_ptr(a) && is_device_ptr(dt) &&
                         (!u || (is_device_ptr(u) && is_device_ptr(dudt)))),
              SPH_E_ARG, "sph_kick_each: arrays must be device memory");
  if (n > 0) LAUNCH(k_kick_each, grid1d(c, n, 256), 256, 0, n, v, u, a, dudt, dt);
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

int sph_timebins(sph_ctx* ctx, int64_t n, const float* h, const float* vsig, float c_cfl, double dt_min,
                 int32_t n_bins, int64_t ti, const uint8_t* active, const int64_t* ticks_in, int32_t cap2,
                 int64_t* ticks_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && (n == 0 || (h && vsig && ticks_out)) && c_cfl > 0.f && dt_min > 0.0 && n_bins >= 0 &&
                  n_bins < 62 && ti >= 0 && (!active || ticks_in),
              SPH_E_ARG, "bad argument");
  const void* ptrs[5] = {h, vsig, ticks_out, active, ticks_in};
  for (int i = 0; i < 5; ++i)
    SPH_REQUIRE(!ptrs[i] || n == 0 || is_device_ptr(ptrs[i]), SPH_E_ARG, "sph_timebins: arrays must be device memory");
  if (n > 0)
    LAUNCH(k_timebins, grid1d(c, n, 256), 256, 0, n, h, vsig, c_cfl, dt_min, n_bins, (long long)ti, active,
           reinterpret_cast<const long long*>(ticks_in), cap2, reinterpret_cast<long long*>(ticks_out));
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

int sph_timebins_wake(sph_ctx* ctx, int64_t n, const uint8_t* active, const float* lim, int64_t ti_end,
                      const int64_t* ti_begin, int64_t* ticks, double dt_min, float* kick) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && (n == 0 || (lim && ti_begin && ticks && kick)) && dt_min > 0.0, SPH_E_ARG, "bad argument");
  const void* ptrs[5] = {active, lim, ti_begin, ticks, kick};
  for (int i = 0; i < 5; ++i)
    SPH_REQUIRE(!ptrs[i] || n == 0 || is_device_ptr(ptrs[i]), SPH_E_ARG,
                "sph_timebins_wake: arrays must be device memory");
  if (n > 0)
    LAUNCH(k_timebins_wake, grid1d(c, n, 256), 256, 0, n, active, lim, (long long)ti_end,
           reinterpret_cast<const long long*>(ti_begin), reinterpret_cast<long long*>(ticks), dt_min, kick);
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

int sph_drift(sph_ctx* ctx, int64_t n, float* x, const float* v, float dt) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n >= 0 && (n == 0 || (x && v)), SPH_E_ARG, "bad argument");
  SPH_REQUIRE(n == 0 || (is_device_ptr(x) && is_device_ptr(v)), SPH_E_ARG, "sph_drift: arrays must be device memory");
  if (n > 0)
    LAUNCH(k_drift, grid1d(c, n, 256), 256, 0, n, x, v, dt, (float)c->cfg.box[0], (float)c->cfg.box[1],
           (float)c->cfg.box[2]);
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

int sph_timestep(sph_ctx* ctx, int64_t n, const float* h, const float* vsig, float c_cfl, float* dt_out,
                 float* dt_min_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n > 0 && h && vsig && dt_min_out && c_cfl > 0.f, SPH_E_ARG, "bad argument");
  SPH_REQUIRE(is_device_ptr(h) && is_device_ptr(vsig) && (!dt_out || is_device_ptr(dt_out)), SPH_E_ARG,
              "sph_timestep: arrays must be device memory");
  unsigned* mb = B<unsigned>(c, B_TSTEP, 1);
  const unsigned inf = 0x7f800000u;
  CUDA_TRY(cudaMemcpyAsync(mb, &inf, sizeof(unsigned), cudaMemcpyHostToDevice, c->stream));
  LAUNCH(k_timestep, grid1d(c, n, 256), 256, 0, n, h, vsig, c_cfl, dt_out, mb);
  unsigned r = 0;
  CUDA_TRY(cudaMemcpyAsync(&r, mb, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  memcpy(dt_min_out, &r, 4);
  API_END
  return SPH_OK;
}

// ------------------------------------------------------------------ NCCL transport ---
// The ring of slabs: rank r exchanges with lower = r - 1 and upper = r + 1
// (mod nranks). Messages to one peer match in posting order, so a rank sends its upper face
// first and receives its lower halo first: with nranks <= 2 (one peer on both sides, or the
// rank itself) the upper face of the lower neighbour still lands in the lower halo.

int sph_comm_unique_id(uint8_t* id_out) {
  if (!id_out) return SPH_E_ARG;
  if (!nccl().ok) return SPH_E_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return SPH_E_NCCL;
  memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return SPH_OK;
}

int sph_comm_init(sph_ctx* ctx, const uint8_t* id) {
  API_BEGIN(ctx)
  SPH_REQUIRE(id != nullptr, SPH_E_ARG, "id == NULL");
  SPH_REQUIRE(c->cfg.nranks >= 1 && c->cfg.rank >= 0 && c->cfg.rank < c->cfg.nranks, SPH_E_ARG,
              "cfg.rank / cfg.nranks out of range");
  SPH_REQUIRE(c->comm == nullptr, SPH_E_STATE, "communicator already initialised");
  SPH_REQUIRE(nccl().ok, SPH_E_NCCL, nccl().why);
  ncclUniqueId uid;
  memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  NCCL_TRY(nccl().CommInitRank(&comm, c->cfg.nranks, uid, c->cfg.rank));
  c->comm = comm;
  API_END
  return SPH_OK;
}

static void ring_exchange(sph_ctx* c, const void* s_lo, size_t n_lo, const void* s_hi, size_t n_hi, void* r_lo,
                          size_t m_lo, void* r_hi, size_t m_hi, ncclDataType_t t) {
  const int P = c->cfg.nranks, r = c->cfg.rank;
  const int lower = (r - 1 + P) % P, upper = (r + 1) % P;
  ncclComm_t comm = (ncclComm_t)c->comm;
  NCCL_TRY(nccl().GroupStart());
  if (n_hi) NCCL_TRY(nccl().Send(s_hi, n_hi, t, upper, comm, c->stream));
  if (n_lo) NCCL_TRY(nccl().Send(s_lo, n_lo, t, lower, comm, c->stream));
  if (m_lo) NCCL_TRY(nccl().Recv(r_lo, m_lo, t, lower, comm, c->stream));
  if (m_hi) NCCL_TRY(nccl().Recv(r_hi, m_hi, t, upper, comm, c->stream));
  NCCL_TRY(nccl().GroupEnd());
}

int sph_halo_counts(sph_ctx* ctx, int64_t n_lo, int64_t n_hi, int64_t* m_lo, int64_t* m_hi) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->comm != nullptr, SPH_E_STATE, "sph_halo_counts before sph_comm_init");
  SPH_REQUIRE(n_lo >= 0 && n_hi >= 0 && m_lo && m_hi, SPH_E_ARG, "bad argument");
  int64_t* d = B<int64_t>(c, B_TMPL0, 4);
  const int64_t h[2] = {n_lo, n_hi};
  CUDA_TRY(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  ring_exchange(c, d, 1, d + 1, 1, d + 2, 1, d + 3, 1, ncclInt64);
  int64_t got[2];
  CUDA_TRY(cudaMemcpyAsync(got, d + 2, sizeof(got), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  *m_lo = got[0];
  *m_hi = got[1];
  API_END
  return SPH_OK;
}

int sph_halo_exchange(sph_ctx* ctx, int32_t cols, const float* send_lo, int64_t n_lo, const float* send_hi,
                      int64_t n_hi, float* recv_lo, int64_t m_lo, float* recv_hi, int64_t m_hi) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->comm != nullptr, SPH_E_STATE, "sph_halo_exchange before sph_comm_init");
  SPH_REQUIRE(cols > 0 && n_lo >= 0 && n_hi >= 0 && m_lo >= 0 && m_hi >= 0, SPH_E_ARG, "bad argument");
  const void* ptrs[4] = {send_lo, send_hi, recv_lo, recv_hi};
  const int64_t cnt[4] = {n_lo, n_hi, m_lo, m_hi};
  for (int k = 0; k < 4; ++k)
    if (cnt[k] > 0)
      SPH_REQUIRE(ptrs[k] && is_device_ptr(ptrs[k]), SPH_E_ARG, "halo buffers must be device memory");
  ring_exchange(c, send_lo, (size_t)n_lo * cols, send_hi, (size_t)n_hi * cols, recv_lo, (size_t)m_lo * cols, recv_hi,
                (size_t)m_hi * cols, ncclFloat32);
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

int sph_allreduce(sph_ctx* ctx, void* buf, int64_t count, int32_t dtype, int32_t op) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->comm != nullptr, SPH_E_STATE, "sph_allreduce before sph_comm_init");
  SPH_REQUIRE(count >= 0 && (dtype == 0 || dtype == 1) && (op == 0 || op == 1), SPH_E_ARG, "bad argument");
  if (count == 0) return SPH_OK;
  SPH_REQUIRE(buf && is_device_ptr(buf), SPH_E_ARG, "buffer must be device memory");
  NCCL_TRY(nccl().AllReduce(buf, buf, (size_t)count, dtype == 0 ? ncclFloat64 : ncclInt64, op == 0 ? ncclSum : ncclMax,
                            (ncclComm_t)c->comm, c->stream));
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}
