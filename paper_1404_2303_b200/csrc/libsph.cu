// libsph.cu — host orchestration and the C ABI declared in include/sph.h.
// One translation unit (unity build) so every kernel is launched from the file that
// defines it; compiled for sm_100a only (see paper_1404_2303_b200/build.py).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <cstdlib>
#include <ctime>

#include "common.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"
#include "build.cuh"
#include "interact.cuh"

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

static void sync(sph_ctx* c) { CUDA_TRY(cudaStreamSynchronize(c->stream)); }

static bool dbg_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPH_DEBUG");
    v = (e && e[0] && e[0] != '0') ? 1 : 0;
  }
  return v == 1;
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

// =========================================================== counters ===========
static unsigned long long* ctr(sph_ctx* c) { return B<unsigned long long>(c, B_COUNTERS, C_NCOUNTERS); }
static void ctr_reset(sph_ctx* c) {
  static const unsigned long long init[C_NCOUNTERS] = {0, 0, 0, 0, 0, 0, 0, 0x7f800000ull};   // C_HMINBITS = +inf
  static_assert(C_HMINBITS == 7, "counter layout");
  CUDA_TRY(cudaMemcpyAsync(ctr(c), init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
}
static void ctr_read(sph_ctx* c, unsigned long long* h) {
  CUDA_TRY(cudaMemcpyAsync(h, ctr(c), sizeof(unsigned long long) * C_NCOUNTERS, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
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
  CUDA_TRY(cudaMemcpyAsync(&total, sums + nb, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  return total;
}

// =========================================================== radix sort =========
static bool g_radix_attr = false;
static void radix_sort(sph_ctx* c, uint64_t*& keys, uint32_t*& vals, uint64_t*& kalt, uint32_t*& valt,
                       int64_t n, int bits) {
  if (n <= 1) return;
  int npass = std::max(1, (bits + 7) / 8);
  SPH_REQUIRE(npass <= 8, SPH_E_ARG, "radix sort: more than 64 key bits");
  SPH_REQUIRE(n < (1ll << 30), SPH_E_ARG, "radix sort: n >= 2^30");
  uint32_t* hist = B<uint32_t>(c, B_SORT_HIST, 16 * 256);
  CUDA_TRY(cudaMemsetAsync(hist, 0, 8 * 256 * sizeof(uint32_t), c->stream));
  LAUNCH(k_radix_hist, grid1d(c, n, 256), 256, 0, keys, n, npass, hist);
  uint32_t h[8 * 256], g[8 * 256];
  CUDA_TRY(cudaMemcpyAsync(h, hist, npass * 256 * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  bool trivial[8];
  for (int p = 0; p < npass; ++p) {
    uint32_t run = 0;
    trivial[p] = false;
    for (int d = 0; d < 256; ++d) {
      g[p * 256 + d] = run;
      run += h[p * 256 + d];
      if (h[p * 256 + d] == (uint32_t)n) trivial[p] = true;
    }
  }
  uint32_t* gofs = hist + 8 * 256;
  CUDA_TRY(cudaMemcpyAsync(gofs, g, npass * 256 * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
  int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  uint32_t* status = B<uint32_t>(c, B_SORT_STATUS, ntiles * 256);
  uint32_t* tctr = B<uint32_t>(c, B_SORT_CTR, 8);
  if (!g_radix_attr) {
    CUDA_TRY(cudaFuncSetAttribute(k_radix_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RadixSmem)));
    g_radix_attr = true;
  }
  CUDA_TRY(cudaMemsetAsync(tctr, 0, 8 * sizeof(uint32_t), c->stream));
  for (int p = 0; p < npass; ++p) {
    if (trivial[p]) continue;
    CUDA_TRY(cudaMemsetAsync(status, 0, ntiles * 256 * sizeof(uint32_t), c->stream));
    LAUNCH(k_radix_pass, (int)ntiles, RS_THREADS, sizeof(RadixSmem), keys, vals, kalt, valt, n, 8 * p,
           gofs + 256 * p, status, tctr + p);
    std::swap(keys, kalt);
    std::swap(vals, valt);
  }
  sync(c);  // the host arrays h/g above are stack buffers used by async copies
}

// =========================================================== nodes ==============
static NodeArrays nodes(sph_ctx* c) {
  NodeArrays N;
  N.first = Bget<int>(c, B_N_FIRST);
  N.count = Bget<int>(c, B_N_COUNT);
  N.ijk = Bget<int4>(c, B_N_IJK);
  N.parent = Bget<int>(c, B_N_PARENT);
  N.child = Bget<int>(c, B_N_CHILD);
  N.hmaxb = Bget<float>(c, B_N_HMAXB);
  N.split = Bget<int>(c, B_N_SPLIT);
  N.slot = Bget<int>(c, B_N_SLOT);
  N.nA = Bget<int>(c, B_N_NA);
  N.nR = Bget<int>(c, B_N_NR);
  N.amask = Bget<int>(c, B_N_AMASK);
  N.rmask = Bget<int>(c, B_N_RMASK);
  N.offA = Bget<int64_t>(c, B_N_OFFA);
  N.offR = Bget<int64_t>(c, B_N_OFFR);
  N.hmaxA = Bget<float>(c, B_N_HMAXA);
  N.hmaxR = Bget<float>(c, B_N_HMAXR);
  return N;
}

static void ensure_nodes(sph_ctx* c, int64_t cap) {
  B<int>(c, B_N_FIRST, cap, true);
  B<int>(c, B_N_COUNT, cap, true);
  B<int4>(c, B_N_IJK, cap, true);
  B<int>(c, B_N_PARENT, cap, true);
  B<int>(c, B_N_CHILD, 8 * cap, true);
  B<float>(c, B_N_HMAXB, cap, true);
  B<int>(c, B_N_SPLIT, cap, true);
}

static LevelGeom level_geom(sph_ctx* c) {
  LevelGeom g;
  memset(&g, 0, sizeof(g));
  for (int l = 0; l <= SPH_MAX_DEPTH + 1; ++l) {
    float hm = 1e30f;
    for (int k = 0; k < 3; ++k) {
      g.E[l][k] = (float)(c->E0[k] / (double)(1 << l));
      g.n[l][k] = c->ntop[k] << std::min(l, 20);
      hm = std::min(hm, (float)(0.5 * c->E0[k] / (double)(1 << l)));
    }
    g.half_min[l] = hm;
  }
  for (int k = 0; k < 3; ++k) g.L[k] = (float)c->cfg.box[k];
  g.depth = c->depth;
  return g;
}

// largest h the cells may be built for: 3 top cells per axis (with rounding slack)
static float hb_cap(sph_ctx* c) {
  double Lmin = std::min(c->cfg.box[0], std::min(c->cfg.box[1], c->cfg.box[2]));
  return (float)(Lmin / (3.0 * c->cfg.top_edge_factor) * (1.0 - 1e-5));
}

static float as_float(unsigned long long b) {
  uint32_t u = (uint32_t)b;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

// =========================================================== build ==============
// Builds the structure for the caller-order state in B_XIN (positions) and B_HB_ORIG
// (h_build), carrying B_HCUR_O / B_LO_O / B_HI_O into cell order. count_only: the
// occupancy-only hierarchy used for the initial guess (no slots, no sorts).
static void build_structure(sph_ctx* c, bool count_only) {
  DbgTimer _t(c, count_only ? "build (count only)" : "build");
  const int64_t n = c->n;
  const float* x = Bget<float>(c, B_XIN);
  float* hb_o = Bget<float>(c, B_HB_ORIG);
  double L[3] = {c->cfg.box[0], c->cfg.box[1], c->cfg.box[2]};
  double Lmin = std::min(L[0], std::min(L[1], L[2]));
  const double V = L[0] * L[1] * L[2];
  double hmax, hmin;
  if (count_only) {
    // top edge from the mean density; depth as deep as the key allows
    hmax = cbrt(3.0 * c->cfg.n_ngb * V / (4.0 * M_PI * (double)n));
    hmin = hmax / 1024.0;
  } else {
    ctr_reset(c);
    LAUNCH(k_hrange, grid1d(c, n, 256), 256, 0, hb_o, n, ctr(c));
    unsigned long long h[C_NCOUNTERS];
    ctr_read(c, h);
    SPH_REQUIRE(!(h[C_ERR] & ERRBIT_H), SPH_E_DOMAIN, "smoothing length negative or non-finite");
    SPH_REQUIRE(h[C_HMAXBITS] != 0, SPH_E_DOMAIN, "all smoothing lengths are zero");
    hmax = as_float(h[C_HMAXBITS]);
    hmin = as_float(h[C_HMINBITS]);
  }
  int64_t ntot = 1;
  for (int k = 0; k < 3; ++k) {
    double nk = floor(L[k] / (c->cfg.top_edge_factor * hmax * (1.0 + 1e-6)));
    if (count_only) nk = std::max(nk, 3.0);
    SPH_REQUIRE(nk >= 3.0, SPH_E_DOMAIN,
                "smoothing length >= L/3: fewer than 3 top cells per axis (h_build max = " +
                    std::to_string(hmax) + ")");
    nk = std::min(nk, 512.0);
    c->ntop[k] = (int)nk;
    c->E0[k] = L[k] / nk;
    ntot *= (int64_t)nk;
  }
  int top_bits = 0;
  while ((1ll << top_bits) < ntot) ++top_bits;
  double emin = std::min(c->E0[0], std::min(c->E0[1], c->E0[2]));
  int depth = count_only ? SPH_MAX_DEPTH : (int)floor(log2(emin / (2.0 * hmin))) + 1;
  depth = std::max(0, std::min(depth, SPH_MAX_DEPTH));
  while (top_bits + 3 * depth > 63) --depth;
  c->depth = depth;
  c->top_bits = top_bits;
  const int kbits = top_bits + 3 * depth;

  // ---- a2 keys + radix sort
  uint64_t* k0 = B<uint64_t>(c, B_KEYS0, n);
  uint64_t* k1 = B<uint64_t>(c, B_KEYS1, n);
  uint32_t* v0 = B<uint32_t>(c, B_VALS0, n);
  uint32_t* v1 = B<uint32_t>(c, B_VALS1, n);
  const double sc[3] = {(double)((int64_t)c->ntop[0] << depth) / L[0], (double)((int64_t)c->ntop[1] << depth) / L[1],
                        (double)((int64_t)c->ntop[2] << depth) / L[2]};
  LAUNCH(k_keys, grid1d(c, n, 256), 256, 0, x, n, c->ntop[0], c->ntop[1], c->ntop[2], depth, sc[0], sc[1], sc[2],
         k0, v0);
  radix_sort(c, k0, v0, k1, v1, n, kbits);
  uint64_t* keys = k0;
  uint32_t* perm = B<uint32_t>(c, B_PERM, n);
  CUDA_TRY(cudaMemcpyAsync(perm, v0, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->stream));

  // ---- a3 cell-order pack
  float4* xh = B<float4>(c, B_XH, n);
  float* hb = B<float>(c, B_HB, n);
  float* lo = B<float>(c, B_HLO, n);
  float* hi = B<float>(c, B_HHI, n);
  LAUNCH(k_gather_build, grid1d(c, n, 256), 256, 0, perm, n, x, Bget<float>(c, B_HCUR_O), hb_o,
         Bget<float>(c, B_LO_O), Bget<float>(c, B_HI_O), xh, hb, lo, hi);

  // ---- a4 hierarchy: level 0 = runs of the top-cell index
  int* flag = B<int>(c, B_TMPI0, n);
  int* idx = B<int>(c, B_TMPI1, n);
  const int sh = 3 * depth;
  LAUNCH(k_mark_top, grid1d(c, n, 256), 256, 0, keys, n, sh, flag);
  int n0 = scan_excl<int>(c, flag, idx, n);
  ensure_nodes(c, std::max<int64_t>(2 * (int64_t)n0 + 1024, n / 16));
  int* topmap = B<int>(c, B_TOPMAP, ntot);
  CUDA_TRY(cudaMemsetAsync(topmap, 0xff, ntot * sizeof(int), c->stream));
  NodeArrays N = nodes(c);
  LAUNCH(k_write_top, grid1d(c, n, 256), 256, 0, keys, n, sh, flag, idx, c->ntop[0], c->ntop[1], N, topmap);
  LAUNCH(k_top_counts, gridfull(n0, 256), 256, 0, n0, n, N);
  c->lev_off.assign({0, n0});
  LevelGeom g = level_geom(c);
  const int split_count = count_only ? 32 : c->cfg.split_count;
  for (int l = 0;; ++l) {
    const int a = c->lev_off[l], b = c->lev_off[l + 1];
    const int nl = b - a;
    int* nch = B<int>(c, B_N_NCH, nl);
    int* chscan = B<int>(c, B_N_CHBASE, nl);
    N = nodes(c);
    LAUNCH(k_level_split, gridfull((int64_t)nl * 32, 256), 256, 0, a, b, l, depth, hb, keys, g.half_min[l],
           split_count, c->cfg.split_fraction, count_only ? 1 : 0, N, nch, N.child);
    int nnext = scan_excl<int>(c, nch, chscan, nl);
    ensure_nodes(c, (int64_t)b + nnext + 1);
    N = nodes(c);
    LAUNCH(k_make_children, gridfull(nl, 256), 256, 0, a, b, (int64_t)b, nch, chscan, N);
    if (nnext == 0) break;
    c->lev_off.push_back(b + nnext);
  }
  c->n_nodes = c->lev_off.back();
  const int nnodes = c->n_nodes;
  const int nlev = (int)c->lev_off.size() - 1;
  if (count_only) return;

  // ---- a5 neighbour slots (27 per node; 13 = self), interaction levels, list sizes
  B<int>(c, B_N_SLOT, 27 * (int64_t)nnodes);
  B<int>(c, B_N_NA, nnodes);
  B<int>(c, B_N_NR, nnodes);
  B<int>(c, B_N_AMASK, nnodes);
  B<int>(c, B_N_RMASK, nnodes);
  B<int64_t>(c, B_N_OFFA, nnodes);
  B<int64_t>(c, B_N_OFFR, nnodes);
  B<float>(c, B_N_HMAXA, nnodes);
  B<float>(c, B_N_HMAXR, nnodes);
  uint8_t* tau = B<uint8_t>(c, B_TAU, n);
  N = nodes(c);
  LAUNCH(k_top_slots, gridfull(n0, 128), 128, 0, n0, c->ntop[0], c->ntop[1], c->ntop[2], topmap, N);
  for (int l = 1; l < nlev; ++l) {
    const int a = c->lev_off[l], b = c->lev_off[l + 1];
    LAUNCH(k_child_slots, gridfull(b - a, 128), 128, 0, a, b, N);
  }
  LAUNCH(k_tau, gridfull((int64_t)nnodes * 32, 256), 256, 0, nnodes, N, g, hb, tau);
  LAUNCH(k_level_counts, gridfull((int64_t)nnodes * 32, 256), 256, 0, nnodes, N, tau);
  int64_t* nsort = B<int64_t>(c, B_N_NSORT, 2 * (int64_t)nnodes);
  int64_t* sscan = B<int64_t>(c, B_TMPL1, 2 * (int64_t)nnodes);
  LAUNCH(k_list_masks, gridfull(nnodes, 128), 128, 0, nnodes, N, c->cfg.sort_min_len, nsort);
  c->n_sorted = scan_excl<int64_t>(c, nsort, sscan, 2 * (int64_t)nnodes);
  LAUNCH(k_split_offsets, gridfull(nnodes, 256), 256, 0, nnodes, sscan, N);

  // ---- a6 13-direction sorted lists (+ the unsorted self copy)
  SortEntry* sorted = B<SortEntry>(c, B_SORTED, c->n_sorted);
  LAUNCH(k_sort_warp, gridfull((int64_t)nnodes * 64, 256), 256, 0, nnodes, xh, tau, N, g, sorted);
  {
    static bool attr = false;
    const int smem = SORT_BLOCK_MAX * (8 + 4 + 4);
    if (!attr) {
      CUDA_TRY(cudaFuncSetAttribute(k_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = true;
    }
    LAUNCH(k_sort_block, 2 * nnodes, 512, smem, nnodes, xh, tau, N, g, sorted);
  }
  {
    const int nseg = 2 * nnodes;
    int* bflag = B<int>(c, B_TASKFLAG, nseg);
    int* bidx = B<int>(c, B_TASKIDX, nseg);
    int64_t* bsz = B<int64_t>(c, B_TMPL0, nseg);
    LAUNCH(k_mark_big, gridfull(nseg, 256), 256, 0, nnodes, N, bflag, bsz);
    int nbig = scan_excl<int>(c, bflag, bidx, nseg);
    if (nbig > 0) {
      int64_t* bscan = B<int64_t>(c, B_TMPL1, nseg);
      int64_t nent = scan_excl<int64_t>(c, bsz, bscan, nseg);
      int* bigseg = B<int>(c, B_BIGNODES, nbig);
      int64_t* bigoff = B<int64_t>(c, B_BIGOFF, nbig);
      LAUNCH(k_compact_big, gridfull(nseg, 256), 256, 0, nseg, bflag, bidx, bscan, bigseg, bigoff);
      uint64_t* bk0 = B<uint64_t>(c, B_KEYS0, nent);
      uint64_t* bk1 = B<uint64_t>(c, B_KEYS1, nent);
      uint32_t* bv0 = B<uint32_t>(c, B_VALS0, nent);
      uint32_t* bv1 = B<uint32_t>(c, B_VALS1, nent);
      N = nodes(c);
      LAUNCH(k_big_keys, nbig, 512, 0, nbig, bigseg, bigoff, xh, tau, N, g, bk0, bv0);
      int segbits = 0;
      while ((1ll << segbits) < (int64_t)nbig * 14) ++segbits;
      radix_sort(c, bk0, bv0, bk1, bv1, nent, 32 + segbits);
      LAUNCH(k_big_write, nbig, 512, 0, nbig, bigseg, bigoff, N, bk0, bv0, sorted);
    }
  }
  {
    int* cnt2 = B<int>(c, B_SEGCNT2, 2 * (int64_t)nnodes);
    int* off2 = B<int>(c, B_SEGOFF2, 2 * (int64_t)nnodes);
    LAUNCH(k_seg_count, gridfull(nnodes, 128), 128, 0, nnodes, N, cnt2);
    const int nseg = scan_excl<int>(c, cnt2, off2, 2 * (int64_t)nnodes);
    SegDesc* seg = B<SegDesc>(c, B_SEGDESC, nseg);
    LAUNCH(k_seg_fill, gridfull(nnodes, 128), 128, 0, nnodes, N, g, off2, seg);
    c->n_pair_slots = nseg;
  }

  // ---- tasks: leaf cells in chunks of <= 32 particles
  int ntasks;
  {
    int* nchunk = B<int>(c, B_TASKFLAG, nnodes);
    int* cscan = B<int>(c, B_TASKIDX, nnodes);
    N = nodes(c);
    LAUNCH(k_leaf_chunks, gridfull(nnodes, 256), 256, 0, nnodes, N, nchunk);
    ntasks = scan_excl<int>(c, nchunk, cscan, nnodes);
    int4* tasks = B<int4>(c, B_TASKS, ntasks);
    LAUNCH(k_write_tasks, gridfull(nnodes, 256), 256, 0, nnodes, N, nchunk, cscan, tasks);
    c->n_leaves = ntasks;   // number of tasks (stats.n_leaves)
  }
  sync(c);
  DBG("build: n %lld top %dx%dx%d depth %d levels %d nodes %d tasks %d sorted %lld big %s\n", (long long)n,
      c->ntop[0], c->ntop[1], c->ntop[2], depth, nlev, nnodes, ntasks, (long long)c->n_sorted, "");
}

// =========================================================== inputs =============
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

static TravParams trav(sph_ctx* c, const int4* tasks, int ntasks, const uint8_t* active) {
  TravParams P;
  P.tasks = tasks;
  P.ntasks = ntasks;
  P.N = nodes(c);
  P.g = level_geom(c);
  P.sorted = Bget<SortEntry>(c, B_SORTED);
  P.tau = Bget<uint8_t>(c, B_TAU);
  P.seg = Bget<SegDesc>(c, B_SEGDESC);
  P.segoff2 = Bget<int>(c, B_SEGOFF2);
  P.segcnt2 = Bget<int>(c, B_SEGCNT2);
  P.active = active;
  float Lmax = (float)std::max(c->cfg.box[0], std::max(c->cfg.box[1], c->cfg.box[2]));
  P.slack = 4e-7f * Lmax;
  {
    const char* e = getenv("SPH_DEBUG_SKIP");
    P.dbg_skip = e ? atoi(e) : 0;
    const char* d = getenv("SPH_DESC_MIN");
    P.desc_min = d ? atoi(d) : 32;
  }
  P.ctr = ctr(c);
  return P;
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
  cfg->sort_min_len = 96;
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
    if (stream) {
      c->stream = (cudaStream_t)stream;
    } else {
      CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    for (int i = 0; i < 12; ++i) CUDA_TRY(cudaEventCreate(&c->ev[i]));
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
  } catch (const SphError& e) {
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
  for (int i = 0; i < 96; ++i) dev_free(c, c->b[i].p);
  if (c->ev_ok)
    for (int i = 0; i < 12; ++i) cudaEventDestroy(c->ev[i]);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return SPH_OK;
}

int sph_set_allocator(sph_ctx* c, void* (*alloc)(size_t, void*, void*), void (*release)(void*, void*, void*),
                      void* user) {
  if (!c) return SPH_E_ARG;
  if ((alloc == nullptr) != (release == nullptr)) return SPH_E_ARG;
  for (int i = 0; i < 96; ++i)
    if (c->b[i].p) return SPH_E_STATE;
  c->ualloc = alloc;
  c->urelease = release;
  c->uuser = user;
  return SPH_OK;
}

int sph_build_cells(sph_ctx* ctx, int64_t n, const float* x, const float* h0) {
  return sph_build_cells_halo(ctx, n, 0, x, h0);
}

int sph_build_cells_halo(sph_ctx* ctx, int64_t n_own, int64_t n_halo, const float* x, const float* h0) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n_own > 0 && n_halo >= 0 && x, SPH_E_ARG, "n_own <= 0, n_halo < 0 or x == NULL");
  const int64_t n = n_own + n_halo;
  SPH_REQUIRE(n < (1ll << 30), SPH_E_ARG, "n >= 2^30");
  c->n = n;
  c->n_own = n_own;
  c->force_ready = false;
  c->state = 0;
  c->rebuilds = 0;
  CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
  float* xd = B<float>(c, B_XIN, 3 * n);
  CUDA_TRY(cudaMemcpyAsync(xd, x, 3 * n * sizeof(float), cudaMemcpyDefault, c->stream));
  ctr_reset(c);
  LAUNCH(k_validate_x, grid1d(c, n, 256), 256, 0, xd, n, (float)c->cfg.box[0], (float)c->cfg.box[1],
         (float)c->cfg.box[2], ctr(c));
  float* hin = B<float>(c, B_HIN, n);
  if (h0) {
    CUDA_TRY(cudaMemcpyAsync(hin, h0, n * sizeof(float), cudaMemcpyDefault, c->stream));
    LAUNCH(k_hrange, grid1d(c, n, 256), 256, 0, hin, n, ctr(c));
    LAUNCH(k_count_zero, grid1d(c, n, 256), 256, 0, hin, n, ctr(c));
  } else {
    CUDA_TRY(cudaMemsetAsync(hin, 0, n * sizeof(float), c->stream));
  }
  unsigned long long hc[C_NCOUNTERS];
  ctr_read(c, hc);
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_NONFINITE), SPH_E_DOMAIN, "non-finite position");
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_XRANGE), SPH_E_DOMAIN, "position outside [0, L)");
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_H), SPH_E_DOMAIN, "h0 negative or non-finite");
  const bool need_guess = !h0 || hc[C_TMP0] > 0;
  float* hcur = B<float>(c, B_HCUR_O, n);
  float* hb = B<float>(c, B_HB_ORIG, n);
  float* lo = B<float>(c, B_LO_O, n);
  float* hi = B<float>(c, B_HI_O, n);
  if (need_guess) {
    // occupancy-only hierarchy -> h from the particle number density of the leaf (or
    // of its first ancestor holding >= n_ngb particles)
    LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, hb, n, 1.0f);
    LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, hcur, n, 1.0f);
    LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, lo, n, 0.0f);
    LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, hi, n, 0.0f);
    build_structure(c, true);
    LevelGeom g = level_geom(c);
    double Lmin = std::min(c->cfg.box[0], std::min(c->cfg.box[1], c->cfg.box[2]));
    LAUNCH(k_guess_h, gridfull(c->n_nodes, 128), 128, 0, c->n_nodes, nodes(c), g, Bget<uint32_t>(c, B_PERM),
           c->cfg.n_ngb, (int)c->cfg.n_ngb, (float)(0.25 * Lmin), hcur);
    if (h0) LAUNCH(k_merge_guess, grid1d(c, n, 256), 256, 0, hin, n, hcur);
    // the occupancy guess is uncertain: bin for a wider margin so the first passes can
    // bracket the root without a rebuild
    LAUNCH(k_init_h, grid1d(c, n, 256), 256, 0, hcur, n, SPH_COLD_MARGIN * c->cfg.h_margin, hb_cap(c), hcur, hb,
           lo, hi);
    c->margin_used = SPH_COLD_MARGIN * c->cfg.h_margin;
  } else {
    LAUNCH(k_init_h, grid1d(c, n, 256), 256, 0, hin, n, c->cfg.h_margin, hb_cap(c), hcur, hb, lo, hi);
    c->margin_used = c->cfg.h_margin;
  }
  build_structure(c, false);
  c->state = 1;
  CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
  if (c->cfg.flags & SPH_F_SYNC) sync(c);
  API_END
  return SPH_OK;
}

static void fill_struct_stats(sph_ctx* c, sph_stats* st) {
  st->n_levels = (int)c->lev_off.size() - 1;
  st->n_cells = c->n_nodes;
  st->n_leaves = c->n_leaves;
  st->n_pair_slots = c->n_pair_slots;
  st->n_rebuilds = c->rebuilds;
}

// re-bin for h_build = h * margin (parked particles: margin_parked), keeping h, its bracket,
// the states and the converged particles' sums (permuted to the new cell order)
static void rebuild_keep_sums(sph_ctx* c, const float* vd, const float* md, const float* ud, float margin_parked,
                              float margin = -1.f) {
  const int64_t n = c->n;
  if (margin < 0.f) margin = c->cfg.h_margin;
  uint8_t* active = Bget<uint8_t>(c, B_FLAG);
  LAUNCH(k_scatter_state, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, Bget<float4>(c, B_XH),
         Bget<float>(c, B_HLO), Bget<float>(c, B_HHI), active, margin, margin_parked, hb_cap(c),
         Bget<float>(c, B_HCUR_O), Bget<float>(c, B_LO_O), Bget<float>(c, B_HI_O), Bget<float>(c, B_HB_ORIG));
  uint8_t* st_o = B<uint8_t>(c, B_STATE_O, n);
  double* sf_o = B<double>(c, B_SF_O, n);
  float4* a0_o = B<float4>(c, B_ACC0_O, n);
  float4* a1_o = B<float4>(c, B_ACC1_O, n);
  LAUNCH(k_scatter_sums, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, active, Bget<double>(c, B_DSUMF),
         Bget<float4>(c, B_DACC0), Bget<float4>(c, B_DACC1), st_o, sf_o, a0_o, a1_o);
  build_structure(c, false);
  c->rebuilds++;
  c->margin_used = margin;
  LAUNCH(k_gather_vmu, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, vd, md, ud, Bget<float4>(c, B_VM),
         Bget<float>(c, B_U));
  LAUNCH(k_gather_sums, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, st_o, sf_o, a0_o, a1_o, active,
         Bget<double>(c, B_DSUMF), Bget<float4>(c, B_DACC0), Bget<float4>(c, B_DACC1));
}

// coarse mode covers any h below the top cell edge (the 27 top cells hold every partner)
static float coarse_cap(sph_ctx* c) {
  double cap = std::min(c->E0[0], std::min(c->E0[1], c->E0[2])) * (1.0 - 1e-5);
  return (float)cap;
}

int sph_density(sph_ctx* ctx, const float* v, const float* m, const float* u, float* h_out, float* rho_out,
                float* omega_out, int32_t* n_nbr_out, float* div_out, float* curl_out, sph_stats* st) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->state >= 1, SPH_E_STATE, "sph_density before sph_build_cells");
  SPH_REQUIRE(v && m && u && h_out && rho_out, SPH_E_ARG, "required pointer is NULL");
  const int64_t n = c->n;
  CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
  // copied: the force loop gathers v and m again after its rebuild
  const float* vd = dev_in(c, v, 3 * n, B_VIN, true);
  const float* md = dev_in(c, m, n, B_MIN, true);
  const float* ud = dev_in(c, u, n, B_UIN, true);
  ctr_reset(c);
  LAUNCH(k_validate_vmu, grid1d(c, n, 256), 256, 0, vd, md, ud, n, ctr(c));
  unsigned long long hc[C_NCOUNTERS];
  ctr_read(c, hc);
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_NONFINITE), SPH_E_DOMAIN, "non-finite velocity");
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_MASS), SPH_E_DOMAIN, "mass <= 0 or non-finite");
  SPH_REQUIRE(!(hc[C_ERR] & ERRBIT_U), SPH_E_DOMAIN, "internal energy <= 0 or non-finite");
  if (!is_device_ptr(v) || !is_device_ptr(m) || !is_device_ptr(u)) sync(c);

  float4* vm = B<float4>(c, B_VM, n);
  float* uc = B<float>(c, B_U, n);
  uint8_t* active = B<uint8_t>(c, B_FLAG, n);
  double* sf = B<double>(c, B_DSUMF, n);
  float4* acc0 = B<float4>(c, B_DACC0, n);
  float4* acc1 = B<float4>(c, B_DACC1, n);
  float* s2 = B<float>(c, B_DSUM2, n);
  LAUNCH(k_gather_vmu, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, vd, md, ud, vm, uc);
  LAUNCH(k_init_state, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, c->n_own, active);

  int iters = 0;
  long long unconv = n;
  long long cand_last = 0;
  long long parked = 0;
  while (true) {
    // every task is launched; warps without an unconverged particle exit at once
    const int ntasks = c->n_leaves;
    const int4* tasks = Bget<int4>(c, B_TASKS);
    // cold start: the first pass evaluates N, N', N'' only (nobody converges at the guess)
    const int nonly = (iters == 0 && c->margin_used > 1.2f * c->cfg.h_margin && c->cfg.max_h_iter > 1) ? 1 : 0;
    ctr_reset(c);
    if (ntasks > 0) {
      DbgTimer _t(c, "density kernel");
      TravParams P = trav(c, tasks, ntasks, active);
      if (iters == 0) CUDA_TRY(cudaEventRecord(c->ev[6], c->stream));
      LAUNCH(k_density, gridfull(ntasks, INTERACT_WARPS), INTERACT_WARPS * 32, 0, P, Bget<float4>(c, B_XH), vm,
             Bget<uint8_t>(c, B_TAU), DensOut{nonly, sf, acc0, acc1, s2});
      if (iters == 0) CUDA_TRY(cudaEventRecord(c->ev[7], c->stream));
    }
    ++iters;
    const bool last = iters >= c->cfg.max_h_iter;
    if (last) {
      ctr_read(c, hc);
      if (iters == 1) cand_last = (long long)hc[C_CAND];
      break;  // sums are at the current h; unconverged particles are reported
    }
    LAUNCH(k_h_update, grid1d(c, n, 256), 256, 0, n, Bget<float4>(c, B_XH), Bget<float>(c, B_HB),
           Bget<float>(c, B_HLO), Bget<float>(c, B_HHI), active, sf, acc0, s2, c->cfg.n_ngb, c->cfg.n_ngb_tol,
           coarse_cap(c), nonly, ctr(c));
    ctr_read(c, hc);
    if (iters == 1) cand_last = (long long)hc[C_CAND];
    parked += (long long)hc[C_REBUILD];
    unconv = (long long)hc[C_UNCONV] + parked;
    DBG("density pass %d: cand %llu seg %llu chunks %llu (max/warp %llu, in heavy warps %llu) -> active %llu "
        "(coarse %llu) parked %lld\n", iters, hc[C_CAND], hc[C_TMP1], hc[C_TMP2], hc[C_MAXCH], hc[C_HEAVY],
        hc[C_UNCONV], hc[C_TMP0], parked);
    if (unconv == 0) break;
    if (iters == 1 && c->margin_used > 1.2f * c->cfg.h_margin) {
      // cold start: the cells were binned for the occupancy guess with a wide margin; one
      // Newton step later h is known to a few per cent, so re-bin for it with the normal margin
      rebuild_keep_sums(c, vd, md, ud, 2.0f * c->cfg.h_margin);
      parked = 0;
      vm = Bget<float4>(c, B_VM);
      continue;
    }
    if (hc[C_UNCONV] == 0 && parked > 0) {
      // every other particle has converged; the parked ones want an h beyond the top cells
      // (coarse_cap): re-bin everything for h_build = h * margin, keep h, its bracket and the
      // converged particles' sums, and continue with the parked ones only
      rebuild_keep_sums(c, vd, md, ud, 2.0f * c->cfg.h_margin);
      parked = 0;
      vm = Bget<float4>(c, B_VM);
    }
  }
  // ghost: finalise and write the caller-order outputs
  std::vector<OutMap> maps;
  GhostOut go;
  const int64_t no = c->n_own;
  go.h = dev_out(c, h_out, no, B_OUT0, maps);
  go.rho = dev_out(c, rho_out, no, B_OUT1, maps);
  go.omega = dev_out(c, omega_out, no, B_OUT2, maps);
  go.nnbr = dev_out(c, n_nbr_out, no, B_OUT3, maps);
  go.div = dev_out(c, div_out, no, B_OUT4, maps);
  go.curl = dev_out(c, curl_out, 3 * no, B_OUT5, maps);
  go.perm = Bget<uint32_t>(c, B_PERM);
  go.n_own = no;
  go.h_o = B<float>(c, B_HFIN_O, n);
  go.g_o = B<float4>(c, B_GST_O, n);
  // particles whose final h exceeds the h their cells were built for (coarse mode)
  ctr_reset(c);
  LAUNCH(k_count_loose, grid1d(c, n, 256), 256, 0, n, Bget<float4>(c, B_XH), Bget<float>(c, B_HB), ctr(c));
  LAUNCH(k_ghost, grid1d(c, n, 256), 256, 0, n, Bget<float4>(c, B_XH), uc, sf, acc0, acc1, c->cfg.gamma,
         c->cfg.balsara_eps, go, ctr(c));
  flush_out(c, maps, c->ev[3]);
  c->state = 2;
  c->force_ready = false;
  int status = (unconv > 0 && iters >= c->cfg.max_h_iter) ? SPH_E_NOCONV : SPH_OK;
  ctr_read(c, hc);
  c->loose = (int64_t)hc[C_TMP0];
  if (c->n > c->n_own && c->cfg.halo_width > 0.0) {
    // every owned particle's partners must be inside the received halo
    ctr_reset(c);
    LAUNCH(k_hrange, grid1d(c, c->n_own, 256), 256, 0, Bget<float>(c, B_HFIN_O), c->n_own, ctr(c));
    unsigned long long hh[C_NCOUNTERS];
    ctr_read(c, hh);
    SPH_REQUIRE(as_float(hh[C_HMAXBITS]) <= c->cfg.halo_width, SPH_E_NOCONV,
                "halo too narrow: an owned h = " + std::to_string(as_float(hh[C_HMAXBITS])) + " exceeds cfg.halo_width");
  }
  {
    if (st) {
      memset(st, 0, sizeof(*st));
      fill_struct_stats(c, st);
      st->n_directed = (int64_t)hc[C_NDIR];
      st->n_candidates = cand_last;
      st->n_candidates_density_full = cand_last;
      st->n_unconverged = status == SPH_E_NOCONV ? unconv : 0;
      st->h_iters = iters;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
      st->ms_build = ms;
      cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
      st->ms_density = ms;
      cudaEventElapsedTime(&ms, c->ev[6], c->ev[7]);
      st->ms_kernel_density_full = ms;
    }
  }
  if (status == SPH_E_NOCONV) {
    c->err = "h iteration did not converge in max_h_iter passes: " + std::to_string(unconv) + " particles";
    return status;
  }
  API_END
  return SPH_OK;
}

// Force-loop structure: the density cells were built for h_build (cold-start margin, or
// below the h of particles that finished in coarse mode) and without the halo particles'
// final h; rebuild once, tight (h_build = h), from the caller-order state, then gather the
// force inputs in the new cell order.
static void prepare_force(sph_ctx* c) {
  const int64_t n = c->n;
  const bool rebuild = c->margin_used > 1.2f * c->cfg.h_margin || c->loose > 0 || c->n > c->n_own;
  if (rebuild) {
    DBG("force: tight rebuild (margin used %.3f, %lld loose, %lld halo)\n", c->margin_used, (long long)c->loose,
        (long long)(c->n - c->n_own));
    LAUNCH(k_force_hb, grid1d(c, n, 256), 256, 0, Bget<float>(c, B_HFIN_O), n, Bget<float>(c, B_HCUR_O),
           Bget<float>(c, B_HB_ORIG));
    build_structure(c, false);
    c->rebuilds++;
    c->margin_used = 1.0f;
  }
  float4* fx = B<float4>(c, B_FX, n);
  float4* fs = B<float4>(c, B_FS, n);
  float4* vm = B<float4>(c, B_VM, n);
  LAUNCH(k_gather_force, grid1d(c, n, 256), 256, 0, Bget<uint32_t>(c, B_PERM), n, Bget<float4>(c, B_XH),
         Bget<float>(c, B_HFIN_O), Bget<float4>(c, B_GST_O), Bget<float>(c, B_VIN), Bget<float>(c, B_MIN), fx, fs, vm);
  LAUNCH(k_node_hmax, gridfull((int64_t)c->n_nodes * 32, 256), 256, 0, c->n_nodes, nodes(c), Bget<float4>(c, B_XH),
         Bget<uint8_t>(c, B_TAU));
  c->force_ready = true;
}

int sph_force(sph_ctx* ctx, float* a_out, float* dudt_out, float* vsig_out, int32_t* n_nbr_force_out,
              sph_stats* st) {
  API_BEGIN(ctx)
  SPH_REQUIRE(c->state >= 2, SPH_E_STATE, "sph_force before sph_density");
  SPH_REQUIRE(a_out && dudt_out, SPH_E_ARG, "required pointer is NULL");
  const int64_t n = c->n, no = c->n_own;
  CUDA_TRY(cudaEventRecord(c->ev[4], c->stream));
  DbgTimer _tf(c, "force call");
  if (!c->force_ready) prepare_force(c);
  std::vector<OutMap> maps;
  ForceOut fo;
  fo.a = dev_out(c, a_out, 3 * no, B_OUT0, maps);
  fo.dudt = dev_out(c, dudt_out, no, B_OUT1, maps);
  fo.vsig = dev_out(c, vsig_out, no, B_OUT2, maps);
  fo.nnbr = dev_out(c, n_nbr_force_out, no, B_OUT3, maps);
  fo.perm = Bget<uint32_t>(c, B_PERM);
  fo.n_own = no;
  ctr_reset(c);
  TravParams P = trav(c, Bget<int4>(c, B_TASKS), c->n_leaves, nullptr);
  CUDA_TRY(cudaEventRecord(c->ev[8], c->stream));
  LAUNCH(k_force, gridfull(c->n_leaves, INTERACT_WARPS), INTERACT_WARPS * 32, 0, P, Bget<float4>(c, B_FX),
         Bget<float4>(c, B_VM), Bget<float4>(c, B_FS), c->cfg.alpha, Bget<uint8_t>(c, B_TAU), fo);
  CUDA_TRY(cudaEventRecord(c->ev[9], c->stream));
  flush_out(c, maps, c->ev[5]);
  if (st || (c->cfg.flags & SPH_F_SYNC)) {
    unsigned long long hc[C_NCOUNTERS];
    ctr_read(c, hc);
    if (st) {
      memset(st, 0, sizeof(*st));
      fill_struct_stats(c, st);
      DBG("force: tasks %d cand %llu seg %llu chunks %llu (max/warp %llu heavy %llu) pairs %llu\n", c->n_leaves,
          hc[C_CAND], hc[C_TMP1], hc[C_TMP2], hc[C_MAXCH], hc[C_HEAVY], hc[C_NFORCE] / 2);
      st->n_pairs = (int64_t)(hc[C_NFORCE] / 2);
      st->n_candidates = (int64_t)hc[C_CAND];
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]);
      st->ms_force = ms;
      cudaEventElapsedTime(&ms, c->ev[8], c->ev[9]);
      st->ms_kernel_force = ms;
    }
  }
  API_END
  return SPH_OK;
}

int sph_guess_h(sph_ctx* ctx, int64_t n, const float* x, float* h_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n > 0 && x && h_out, SPH_E_ARG, "bad argument");
  c->n = n;
  c->n_own = n;
  c->state = 0;
  float* xd = B<float>(c, B_XIN, 3 * n);
  CUDA_TRY(cudaMemcpyAsync(xd, x, 3 * n * sizeof(float), cudaMemcpyDefault, c->stream));
  float* hb = B<float>(c, B_HB_ORIG, n);
  float* hcur = B<float>(c, B_HCUR_O, n);
  float* lo = B<float>(c, B_LO_O, n);
  float* hi = B<float>(c, B_HI_O, n);
  LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, hb, n, 1.0f);
  LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, hcur, n, 1.0f);
  LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, lo, n, 0.0f);
  LAUNCH(k_fill_f, grid1d(c, n, 256), 256, 0, hi, n, 0.0f);
  build_structure(c, true);
  double Lmin = std::min(c->cfg.box[0], std::min(c->cfg.box[1], c->cfg.box[2]));
  std::vector<OutMap> maps;
  float* o = dev_out(c, h_out, n, B_OUT0, maps);
  LAUNCH(k_guess_h, gridfull(c->n_nodes, 128), 128, 0, c->n_nodes, nodes(c), level_geom(c), Bget<uint32_t>(c, B_PERM),
         c->cfg.n_ngb, (int)c->cfg.n_ngb, (float)(0.25 * Lmin), o);
  flush_out(c, maps, c->ev[10]);
  sync(c);
  API_END
  return SPH_OK;
}

int sph_halo_select(sph_ctx* ctx, int64_t n, const float* x, double lo, double hi, double width,
                    int32_t* idx_lo_out, int32_t* idx_hi_out, int64_t* counts_out) {
  API_BEGIN(ctx)
  SPH_REQUIRE(n > 0 && x && idx_lo_out && idx_hi_out && counts_out, SPH_E_ARG, "bad argument");
  SPH_REQUIRE(hi > lo && width > 0.0, SPH_E_ARG, "need hi > lo and width > 0");
  const float* xd = dev_in(c, x, 3 * n, B_XIN);
  int* flo = B<int>(c, B_TMPI0, n);
  int* fhi = B<int>(c, B_TMPI1, n);
  int* slo = B<int>(c, B_TASKFLAG, n);
  int* shi = B<int>(c, B_TASKIDX, n);
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
  c->force_ready = false;
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
