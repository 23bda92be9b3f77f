// common.cuh — shared device helpers and the context struct of libsph (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <string>
#include <vector>

#include "../../include/sph.h"

#define SPH_WARP 32
#define FULL_MASK 0xffffffffu

// ---------------------------------------------------------------- errors -----
struct SphError {
  int status;
  std::string msg;
};

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      throw SphError{_e == cudaErrorMemoryAllocation ? SPH_E_OOM : SPH_E_CUDA,        \
                     std::string(#expr) + ": " + cudaGetErrorString(_e)};           \
  } while (0)

#define SPH_REQUIRE(cond, status, msg)                                              \
  do {                                                                              \
    if (!(cond)) throw SphError{(status), (msg)};                                   \
  } while (0)

// ---------------------------------------------------------------- device -----
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}
__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// orderable uint for a float (monotone: a < b <=> ord(a) < ord(b))
__device__ __forceinline__ uint32_t float_ord(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// ---------------------------------------------------------------- packed fp32 -
// sm_100 packed FP32 (FADD2 / FMUL2 / FFMA2): two candidate sources per instruction in the
// distance tests. The operation order of the scalar r^2 = fma(dx, dx, fma(dy, dy, dz*dz)) is
// kept, so the packed test and the interaction body agree bit for bit.
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
// r^2 of two sources (x, y, z pairs) from one target (xi, yi, zi)
__device__ __forceinline__ float2 r2_pair(float xi, float yi, float zi, float2 x, float2 y, float2 z) {
  unsigned long long dx, dy, dz, r;
  const unsigned long long X = f2u(make_float2(xi, xi)), Y = f2u(make_float2(yi, yi)), Z = f2u(make_float2(zi, zi));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(X), "l"(f2u(x)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(Y), "l"(f2u(y)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(Z), "l"(f2u(z)));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(dz));
  asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r) : "l"(dy));
  asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r) : "l"(dx));
  return u2f(r);
}

// ---------------------------------------------------------------- geometry ---
// 27 neighbour offsets o in {-1,0,1}^3, index k = (ox+1)*9 + (oy+1)*3 + (oz+1); k = 13 is
// the cell itself. The 13 canonical sort directions are the offsets whose first non-zero
// component is positive (k = 14..26); offset k < 13 is the flip of 26-k.
__host__ __device__ __forceinline__ int off_x(int k) { return k / 9 - 1; }
__host__ __device__ __forceinline__ int off_y(int k) { return (k / 3) % 3 - 1; }
__host__ __device__ __forceinline__ int off_z(int k) { return k % 3 - 1; }
__host__ __device__ __forceinline__ int slot_dir(int k) { return k > 13 ? k - 14 : 12 - k; }
__host__ __device__ __forceinline__ bool slot_flip(int k) { return k < 13; }

// unit vectors of the 13 canonical directions d (offset k = d + 14), computed on the host
// once (sph_dirs_init) so every kernel uses bit-identical values
__constant__ float c_dirs[14][3];
__device__ __forceinline__ float3 dir_unit(int d) { return make_float3(c_dirs[d][0], c_dirs[d][1], c_dirs[d][2]); }

// ---------------------------------------------------------------- constants --
#define SPH_PI_F 3.14159265358979323846f
#define SPH_CNORM (8.0f / SPH_PI_F)   // 8/pi of W
#define SPH_MAX_DEPTH 12              // Morton levels below the top grid
#define SPH_COLD_MARGIN 1.2f   // h_build / guess at a cold start (C4: 1.0 7.85, 1.1 7.77, 1.2 7.69, 1.3 7.88 ms; C3 flat: tools/cold_margin_sweep.sh)
#ifndef SPH_REGROW_MARGIN
#define SPH_REGROW_MARGIN 1.1f        // h_build / h after a Newton step left the list (tuned: tools/sweep.sh)
#endif
#define SPH_BAND 1e-6f   // borderline band |r/h - 1| <= 1e-6 (north_star; R5)
#define SPH_IDX_BITS 27               // list entry = (periodic image code << 27) | source index
#define SPH_IDX_MASK ((1u << SPH_IDX_BITS) - 1u)
#ifndef SPH_GROUP
#define SPH_GROUP 32                  // targets per group (one warp, one lane per target; <= 32)
#endif
static_assert(SPH_GROUP >= 1 && SPH_GROUP <= 32, "a target group is one warp: 1 <= SPH_GROUP <= 32");

// ---------------------------------------------------------------- context ----
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct sph_ctx {
  sph_config cfg;
  // page-locked scratch for the small device -> host reads (counters, scan totals), so each
  // is one stream-ordered copy + sync instead of a staged pageable copy
  unsigned long long* hpin = nullptr;
  bool ctr_init_ready = false;   // B_CTRINIT holds the counters' initial values
  // sph_step: v, m, u staged on the side stream before the build (pre_in: the caller's
  // pointers, pre_dev: their device views), and the density's host outputs copied on the side
  // stream while the force loop runs (defer_out)
  const float* pre_in[3] = {nullptr, nullptr, nullptr};
  const float* pre_dev[3] = {nullptr, nullptr, nullptr};
  bool pre_pending = false, pre_ready = false, pre_side = false, defer_out = false;
  // CUDA IPC (peer-store halo): buffers this context exposes, buffers of other processes it
  // opened, and interprocess events (created here or opened from a handle)
  std::vector<void*> ipc_own, ipc_open;
  std::vector<cudaEvent_t> ipc_ev;
  void* comm = nullptr;   // ncclComm_t of the slab decomposition (sph_comm_init), or null
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* (*ualloc)(size_t, void*, void*) = nullptr;
  void (*urelease)(void*, void*, void*) = nullptr;
  void* uuser = nullptr;
  std::string err;
  int64_t launches = 0;
  int num_sms = 148;

  int64_t n = 0;        // particles in the structure: owned + halo
  int64_t n_own = 0;    // owned (targets); caller indices >= n_own are halo (sources only)
  int state = 0;        // 0 nothing, 1 cells built, 2 density done, 3 force inputs gathered
  bool force_lists = false;
  // groups with re-walking particles, appended by the walk's solve epilogue (double buffered:
  // rg_cur is the list the next re-walk reads); invalid after a solve outside a walk
  int rg_cur = 0;
  bool has_active = false;   // sph_set_active: a caller-order mask in B_ACTIVE applies to the next build
  int64_t n_active_for = 0;
  float skin = 0.f;            // drift since the cells were sorted (sph_update_cells)
  bool cells_reused = false;
  bool rg_valid = false;
  bool cold = false;       // h0 was the occupancy guess (wider list margin, N-only first pass)

  // geometry of the current structure (built once per sph_build_cells)
  int ntop[3] = {0, 0, 0};
  double E0[3] = {0, 0, 0};
  int depth = 0;             // Morton levels below top (keys carry 3*depth bits)
  int top_bits = 0;
  std::vector<int> lev_off;  // node index offsets per level (size nlevels+1)
  int n_nodes = 0, n_leaves = 0, n_groups = 0;
  int64_t n_sorted = 0;      // entries of all 13-direction lists
  int64_t pool = 0;          // entries of the interaction (UNION) lists
  float cold_margin = SPH_COLD_MARGIN, regrow_margin = SPH_REGROW_MARGIN;
  int nb_k = 192;            // capacity of a particle's neighbour list (NB walk)
  int64_t nb_k_for = -1;     // particle count nb_k was sized for
  int ucap = 768;            // capacity of a group's interaction list slab (UNION walk)
  bool xref_valid = false;   // B_XREF holds the last build's cell-order positions (sph_update_cells)
  bool in_step = false;      // sph_build_cells called by sph_step (no end-of-call sync)
  bool pos_check = false;    // k_keys' position checks not read yet (read with the level build's status)
  int n_groups_lev = -1;     // groups counted by the last level build (-1: not counted)
  bool maybe_presort = true; // some leaf of the last level build qualifies for presorted lists
  int group_cmax = 512;      // targets: balanced chunks of the deepest cells holding <= 512 (0: sibling packing)
  int64_t ovf_used = 0;      // entries of the neighbour-list overflow pool
  int64_t n_ovfidx = 0;      // particles that have a list in the pool (k_hsolve_pool)
  int64_t list_rebuilds = 0; // groups re-walked for a particle whose h outgrew its list
  float hb_max = 0.f;        // largest h_build (density reach)

  // phase timing: event pairs around kernel launches, resolved when the call syncs
  struct Timed {
    cudaEvent_t a, b;
    int phase;
  };
  std::vector<Timed> timed;
  size_t timed_used = 0;
  double ms_phase[4] = {0, 0, 0, 0};   // 0 NB walks, 1 h solve, 2 union walks, 3 binning + sort
  int sort_bits = 0, sort_passes = 0;
  const float* xin = nullptr;   // this call's positions (caller's device array or a staged copy)
  const float* hin = nullptr;   // this call's h0 (or null)
  int64_t nb_entries = 0, walk_launches = 0, h_evals = 0;
  double h_own_max = 0.0;   // largest owned h of the last density call (sph_halo_required)

  // named device buffers
  DBuf b[96];
  cudaEvent_t ev[12];
  cudaStream_t stream2 = nullptr;   // side stream: host->device copies overlapped with the h iteration
  cudaEvent_t ev_side[6];   // [0] side stream may start, [1] v, m, u copied, [2] h ready, [3] h copied back,
                            // [4] v, m, u may be read, [5] v, m, u checked and in cell order
  bool ev_ok = false;
};

enum BufId {
  // caller-order inputs / outputs kept between calls
  B_XIN = 0, B_HIN, B_VIN, B_MIN, B_UIN, B_HFIN_O, B_GST_O,
  // sort scratch
  B_KEYS0, B_KEYS1, B_VALS0, B_VALS1, B_SORT_HIST, B_SORT_STATUS, B_SORT_CTR, B_SCAN_TMP, B_XC,
  // cell-order particle arrays
  B_PERM, B_XH, B_VM, B_U, B_HB, B_HLO, B_HHI, B_STATE, B_DSUMF, B_DACC0, B_DACC1, B_DSUM2,
  B_FX, B_FS,
  // nodes
  B_N_FIRST, B_N_COUNT, B_N_IJK, B_N_PARENT, B_N_CHILD, B_N_SPLIT, B_N_HMAX, B_N_SORTOFF, B_N_REC, B_N_NCH, B_N_CHBASE, B_N_LEV,
  B_TOPMAP,
  // 13-direction sorted lists
  B_SORTED,
  // groups and interaction lists
  B_GROUPS, B_GOFF, B_GLEN, B_LIST, B_NBR2, B_NBCNT, B_NBOFF, B_NBOVF, B_OVFIDX, B_NBENT, B_GKEYS, B_GORDER, B_SHRUNK, B_OVFC, B_OVFCNT, B_HCTR, B_RGL, B_RGCNT, B_XREF, B_TGT, B_ACTIVE, B_TSTEP, B_WALKRAW, B_GFLAG, B_GSEL, B_HRCH,
  // misc scratch
  B_ABLIST, B_WIN, B_CTRINIT, B_VERR, B_PGROUP, B_SYM_IA, B_SYM_IVS, B_SYM_ICNT, B_SYM_JA, B_SYM_JVS, B_SYM_JCNT,
  B_TMPI0, B_TMPI1, B_TMPL0, B_TMPL1, B_COUNTERS, B_OUT0, B_OUT1, B_OUT2, B_OUT3, B_OUT4, B_OUT5,
  B_FOUT0, B_FOUT1, B_FOUT2, B_FOUT3,
  B_COUNT
};
static_assert(B_COUNT <= 96, "too many buffers");

// device counters layout (int64 slots in B_COUNTERS)
enum CounterId {
  C_ERR = 0,        // error bits (validation)
  C_UNCONV,         // unconverged particles after an h update
  C_REGROW,         // particles whose h outgrew their list reach (group list rebuild)
  C_CAND,           // candidate distance tests (lane tests against staged sources)
  C_NDIR,           // D
  C_NFORCE,         // sum of force neighbour counts (2F)
  C_HMAXBITS,       // max h (float bits as int)
  C_HMINBITS,       // min positive h (float bits)
  C_TMP0, C_TMP1, C_TMP2,
  C_BORDER_D,       // SPH_F_DIAGNOSTICS: borderline directed density pairs
  C_BORDER_F,       //   borderline directed force pairs
  C_COINC,          //   coincident directed pairs (r = 0, j != i)
  C_NCOUNTERS
};

#define ERRBIT_NONFINITE 1
#define ERRBIT_XRANGE 2
#define ERRBIT_MASS 4
#define ERRBIT_U 8
#define ERRBIT_H 16
