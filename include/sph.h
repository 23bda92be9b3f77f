/*
 * sph.h — C ABI of libsph: the B200 (sm_100a) hot path of Gonnet's SPH method
 * (arXiv:1404.2303): neighbour finding over a hierarchical cell decomposition
 * with sorted pair interactions, the density loop with h solved to a target
 * neighbour number, and the symmetric pressure + viscosity force loop.
 *
 * Citations: P:<line> = PAPER.md line (section / equation named); R<n> = the
 * readings of the paper listed in DESIGN.md ("Readings").
 *
 * ---------------------------------------------------------------------------
 * Conventions (apply to every call)
 *  - Particle arrays are fp32 unless stated, length n, vectors row-major [n][3],
 *    in the CALLER's particle order. A pointer may be a CUDA device pointer or a
 *    host pointer (pinned or pageable); libsph detects which with
 *    cudaPointerGetAttributes and copies host data in/out itself on the
 *    context's stream.
 *  - Ownership: the caller owns every array it passes; libsph never frees or
 *    keeps them beyond the call. libsph owns everything inside sph_ctx
 *    (cell-ordered copies, cell hierarchy, interaction slots, sorted lists,
 *    scratch) and frees it in sph_destroy.
 *  - Ordering: calls are ordered on the context's stream. With SPH_F_SYNC
 *    (default) each call synchronises before returning, so the status reflects
 *    device errors and the stats are filled.
 *  - Errors: every call returns an sph_status; sph_last_error(ctx) gives the
 *    detail of the last failing call on that context. On error the outputs are
 *    unspecified, except SPH_E_NOCONV, which writes every output from the last
 *    iterate.
 *  - Threads: one context per host thread at a time; distinct contexts are
 *    independent.
 * ---------------------------------------------------------------------------
 */
#ifndef SPH_H
#define SPH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_ABI_VERSION 2

typedef struct sph_ctx sph_ctx;

typedef enum {
  SPH_OK = 0,
  SPH_E_ARG = -1,    /* null required pointer, n <= 0, n changed between calls, bad config
                        (box <= 0, gamma <= 1, alpha < 0, n_ngb <= 32/3, tol <= 0,
                        top_edge_factor < 1, split_fraction outside [0,1)) */
  SPH_E_DOMAIN = -2, /* non-finite input; x outside [0,L); m <= 0; u <= 0; h0 < 0;
                        a smoothing length >= min(L)/2 (minimum image) */
  SPH_E_STATE = -3,  /* order violated: density before build_cells, force before density */
  SPH_E_NOCONV = -4, /* h iteration did not converge: it hit max_h_iter, Eq. 3 has no root for a
                        particle (more than 4 coincident particles, or too few within L/2: R24),
                        or the density loop's re-check of N(h) failed (R4); every output is
                        written (finite) from the last iterate; stats.n_unconverged counts them */
  SPH_E_CUDA = -5,
  SPH_E_NCCL = -6,
  SPH_E_OOM = -7
} sph_status;

/* flags */
#define SPH_F_SYNC 1u             /* synchronise at the end of each call (default on) */
#define SPH_F_COUNT_CANDIDATES 2u /* count distance tests (stats.n_candidates) */
#define SPH_F_DIAGNOSTICS 4u      /* count borderline and coincident pairs (stats.n_borderline,
                                     n_borderline_force, n_coincident) */
#define SPH_F_SYMMETRIC 8u        /* sph_force evaluates every unordered pair once and updates both
                                     particles (j side by shared-memory then global float
                                     reductions: not bitwise deterministic). Default: gather form,
                                     every pair from both sides, deterministic */

typedef struct {
  int32_t abi_version;   /* = SPH_ABI_VERSION */
  double box[3];         /* periodic domain [0,Lx)x[0,Ly)x[0,Lz) */
  float gamma;           /* polytropic index, 5/3 */
  float n_ngb;           /* target weighted neighbour number of Eq. 3, 48 (P:176-182,
                            P:1352); the self term is included (R2) */
  float n_ngb_tol;       /* the iteration stops when |N_i - n_ngb| <= tol, when the bracket is at
                            fp32 resolution of h, or after a Halley step of |d ln h| <= 3e-3 inside
                            the bracket (its residual is ~1e-7 N, R4); the density loop then
                            re-checks every particle with its own sums at the final h and reports
                            |N_i - n_ngb| > 2 tol + 24 n_ngb eps_fp32 as unconverged
                            (SPH_E_NOCONV): the enforced bound is that one (3.4e-4 at the 1e-4
                            default; measured worst case 1.06e-4 on C4). 1.0 = the paper's
                            "e.g. +-1" */
  int32_t max_h_iter;    /* density passes allowed for the h iteration (default 64) */
  float alpha;           /* viscosity alpha, 0.8; 0 disables viscosity */
  float balsara_eps;     /* 1e-4 in the Balsara denominator (R10) */
  int32_t split_count;   /* split a cell only if it holds more particles: 300 */
  float split_fraction;  /* ... and more than this fraction has h < edge/2: 0.875 */
  float top_edge_factor; /* kappa >= 1: top cell edge >= kappa * max h ("larger or equal") */
  float h_margin;        /* >= 1: neighbour lists are recorded for h_build = h * h_margin so the
                            Newton iteration can grow h without a new walk */
  int32_t sort_min_len;  /* leaves holding more particles than this are presorted along the 13
                            pair directions and swept with the windowed early exit;
                            smaller leaves are streamed whole through the box and distance
                            filters. 0 = presort every leaf */
  uint32_t flags;        /* SPH_F_* */
  int32_t rank, nranks;  /* 0, 1 for a single GPU */
  double slab_lo, slab_hi; /* owned x-range of this rank (multi-GPU) */
  double halo_width;     /* multi-GPU: width of the halo received at each slab face; an owned
                            particle within h of a face with h beyond it cannot be evaluated
                            (SPH_E_NOCONV "halo too narrow"; sph_halo_required). 0 = none */
  /* capacities and tuning of the neighbour-finding structures (results do not depend on them) */
  int32_t row_cap;       /* entries of a particle's neighbour row (the h iteration's distances);
                            longer rows shrink h_build once, then go to an exactly sized pool.
                            0 = sized from free device memory (<= 1024) */
  int32_t list_cap;      /* interaction-list slab entries per target group; longer lists are walked
                            again into exactly sized space. 0 = 768 */
  int32_t group_container; /* target groups: chunks of <= 32 consecutive particles of the deepest
                            cells holding <= group_container particles. 0 = 512; -1 = pack sibling
                            leaves instead */
  float cold_margin;     /* h0 == 0 (library guess): rows are recorded for h_build = guess x this.
                            0 = 1.2 */
} sph_config;

typedef struct {         /* host struct, filled when non-NULL */
  int64_t n_pairs;       /* F: unordered pairs with r < max(h_i,h_j) */
  int64_t n_directed;    /* D: ordered (i,j), j != i, r_ij < h_i */
  int64_t n_candidates;  /* distance tests of the last density pass and the force pass
                            (SPH_F_COUNT_CANDIDATES) */
  int64_t n_unconverged; /* particles not converged when the density call returned */
  int64_t n_rebuilds;    /* target groups re-walked because an h outgrew its neighbour list */
  int32_t h_iters;       /* largest number of Newton/Halley iterations of one particle */
  int32_t n_levels;      /* depth of the cell hierarchy + 1 */
  int64_t n_cells, n_leaves, n_pair_slots; /* cells; target groups; interaction-list entries */
  double ms_build, ms_density, ms_force, ms_halo; /* whole calls (CUDA events on the ctx stream) */
  int64_t halo_sent, halo_recv;
  /* kernel-only times (CUDA events bracketing the single launch on the ctx stream) */
  double ms_kernel_density_full; /* the density-sum kernel at the final h (one launch) */
  double ms_kernel_force;        /* the force kernel */
  int64_t n_candidates_density_full; /* distance tests of that density-sum launch */
  /* per-phase kernel time (CUDA events around each launch, summed over launches) */
  double ms_kernel_walk_nb;      /* neighbour-list walks (build + re-walks of the h iteration) */
  double ms_kernel_hsolve;       /* the per-particle h iteration */
  double ms_kernel_walk_union;   /* interaction-list walks */
  int64_t n_nb_entries;          /* neighbour-list entries recorded (all walks) */
  int64_t n_walk_launches;       /* neighbour-list walk launches */
  /* SPH_F_DIAGNOSTICS only (else 0), from the final density and force loops in fp32: */
  int64_t n_borderline;          /* density (sph_density): directed (i, j), j != i, |r_ij/h_i - 1| <= 1e-6 (R5) */
  int64_t n_borderline_force;    /* force (sph_force): unordered pairs, |r_ij/max(h_i,h_j) - 1| <= 1e-6 */
  int64_t n_coincident;          /* density (sph_density): unordered pairs with r_ij = 0, i != j (R13) */
  /* SPH_F_COUNT_CANDIDATES only (else 0), sph_density: sources the walks streamed through their
     box filters (after the sorted windows where leaves are presorted) */
  int64_t n_nb_sources;          /* neighbour-list walks since the last build (incl. re-walks) */
  int64_t n_union_sources;       /* interaction-list walks of this call */
  int32_t cells_reused;          /* 1 if the last build kept the cells (sph_update_cells) */
  /* binning + sort of the last build (a1-a3): keys, radix passes, permute + pack */
  double ms_kernel_sort;         /* CUDA events around those launches */
  int32_t sort_key_bits;         /* top-cell index bits + 3 x Morton levels */
  int32_t sort_passes;           /* 8-bit radix passes */
  /* sph_density: neighbour-list entries summed by the h iteration, over every evaluation of
     N(h) and its derivatives (Eq. 3; the build's fused solve and all re-walk rounds) */
  int64_t n_h_evals;
} sph_stats;

/* Fill *cfg with the paper's defaults for the given box. */
void sph_config_default(sph_config* cfg, double lx, double ly, double lz);

/* Create a context on `cuda_device`, ordered on `cuda_stream` (cudaStream_t or NULL for
 * a context-owned stream). Validates *cfg (SPH_E_ARG). *out is NULL on failure. */
int sph_create(const sph_config* cfg, int cuda_device, void* cuda_stream, sph_ctx** out);
int sph_destroy(sph_ctx* ctx);

/* Route libsph's device allocations through the caller's allocator (e.g. torch's
 * caching allocator). Must be called before the first build. NULL restores cudaMalloc. */
int sph_set_allocator(sph_ctx* ctx, void* (*alloc)(size_t bytes, void* stream, void* user),
                      void (*release)(void* ptr, void* stream, void* user), void* user);

const char* sph_status_string(int status);
const char* sph_last_error(const sph_ctx* ctx);

/* 1. Neighbour-finding structure (section 3.2).
 *    x  [n][3]: positions in [0,L) (copied).
 *    h0 [n] or NULL: initial smoothing lengths (support radius); NULL or
 *       h0[i] == 0 -> library guess from cell occupancy.
 *    Sorts the particles by cell key (top grid with edge >= kappa * max h0, P:471-474,
 *    Morton octants below; device radix sort), splits cells recursively (P:510-518 with
 *    split_count / split_fraction), presorts the leaves longer than sort_min_len along the
 *    13 pair directions, groups the particles into warp-sized target groups and
 *    records every particle's neighbour list (r^2 < h_build^2, h_build = h0 * margin) by a
 *    walk of the hierarchy with the sorted sweeps.
 *    Errors: SPH_E_ARG, SPH_E_DOMAIN (non-finite x, x outside [0,L), h0 < 0 or
 *    h0 >= min(L)/2), SPH_E_CUDA, SPH_E_OOM. At most 2^27 particles per context. */
int sph_build_cells(sph_ctx* ctx, int64_t n, const float* x, const float* h0);

/* 2. Density loop (Eq. 2-3) with h_i solved to N_i = n_ngb +- tol by a
 *    bracketed Newton/Halley iteration (R3-R4) on each particle's recorded
 *    neighbour list (run inside the build's walk; particles whose root lies beyond their
 *    list are re-walked with a larger h_build). Then the sums of Eq. 2 at the final h over
 *    the interaction lists (reach
 *    max(h_i, h_j)) and the "ghost" step: Omega, P, c,
 *    A = P/(Omega rho^2), div/curl v and Balsara f, kept inside ctx.
 *    v [n][3], m [n] (> 0), u [n] (> 0): copied.
 *    Outputs (caller order): h_out [n], rho_out [n]; optional (NULL to skip)
 *    omega_out [n], n_nbr_out [n] (#{j != i : r_ij < h_i}, R21), div_out [n],
 *    curl_out [n][3].
 *    Errors: SPH_E_STATE (no build), SPH_E_DOMAIN, SPH_E_NOCONV, SPH_E_CUDA. */
int sph_density(sph_ctx* ctx, const float* v, const float* m, const float* u,
                float* h_out, float* rho_out, float* omega_out, int32_t* n_nbr_out,
                float* div_out, float* curl_out, sph_stats* st);

/* 3. Force loop: Eq. 4 and Eq. 5 + Monaghan-Balsara viscosity
 *     over every pair with r_ij < max(h_i, h_j), using the
 *    ctx's state from sph_density. Idempotent.
 *    Outputs (caller order): a_out [n][3] (dv/dt), dudt_out [n]; optional
 *    vsig_out [n] (max_j c_i + c_j - 3 w_ij, the Eq. 6 denominator P:1267),
 *    n_nbr_force_out [n] (#{j != i : r_ij < max(h_i,h_j)}).
 *    Errors: SPH_E_STATE (no density), SPH_E_CUDA. */
int sph_force(sph_ctx* ctx, float* a_out, float* dudt_out, float* vsig_out,
              int32_t* n_nbr_force_out, sph_stats* st);

/* ---- multi-GPU slab decomposition (the paper's proxy cells).
 * One process and one context per GPU; each rank owns the particles with x in its slab
 * [lo, hi). The transport (NCCL point-to-point over NVLink) is either libsph's own
 * (sph_comm_init, sph_halo_exchange below) or the caller's, e.g. torch.distributed
 * (paper_1404_2303_b200/slab.py); the other calls do the device work.
 * Sequence per evaluation: sph_halo_select -> exchange x, v, m, u (+h0) of the selected
 * particles -> sph_build_cells_halo -> sph_density -> sph_export_state of the selected
 * particles -> exchange -> sph_import_halo_state -> sph_force. */

/* Owned particles (caller indices 0..n_own-1, the targets) followed by n_halo halo
 * particles (sources only: no outputs, never iterated). x [n_own+n_halo][3], h0 likewise or
 * NULL. Subsequent sph_density inputs v, m, u cover all n_own+n_halo particles; all outputs
 * of sph_density / sph_force cover the owned particles only. */
int sph_build_cells_halo(sph_ctx* ctx, int64_t n_own, int64_t n_halo, const float* x, const float* h0);

/* One whole evaluation, sph_build_cells(n, x, h0) + sph_density(v, m, u, h_out, rho_out) +
 * sph_force(a_out, dudt_out), with the host <-> device copies of host arrays overlapped with
 * the work: v, m, u are copied up on a side stream while the cells and neighbour lists are
 * built, and h, rho come down on the side stream while the force loop runs (page-locked host
 * arrays make these copies asynchronous). Same results, statuses and stats as the three calls;
 * every output is complete on return. st_density / st_force may be NULL. */
int sph_step(sph_ctx* ctx, int64_t n, const float* x, const float* h0, const float* v, const float* m,
             const float* u, float* h_out, float* rho_out, float* a_out, float* dudt_out, sph_stats* st_density,
             sph_stats* st_force);

/* The library's initial guess of h from cell occupancy (the one sph_build_cells uses when
 * h0 is NULL), h_out [n]: N_ngb = (4 pi/3) n h^3 for the local number density n of the
 * smallest cell around the particle holding >= N_ngb particles. Used e.g. to size halos. */
int sph_guess_h(sph_ctx* ctx, int64_t n, const float* x, float* h_out);

/* Indices (ascending, caller order) of the particles within `width` of the lower face
 * (x - lo < width) and of the upper face (hi - x < width) of the slab [lo, hi).
 * idx_lo_out / idx_hi_out have room for n entries; counts_out[0..1] = their lengths. */
int sph_halo_select(sph_ctx* ctx, int64_t n, const float* x, double lo, double hi, double width,
                    int32_t* idx_lo_out, int32_t* idx_hi_out, int64_t* counts_out);

/* The rows sent in the first halo exchange, in one kernel: out [k][9] = {x, y, z, vx, vy, vz, m,
 * u, h0} of the owned particles idx [k] (caller order, as returned by sph_halo_select; h0 may be
 * NULL: 0). All device arrays. */
int sph_halo_pack(sph_ctx* ctx, const float* x, const float* v, const float* m, const float* u, const float* h0,
                  int64_t k, const int32_t* idx, float* out);

/* After sph_density: per listed owned particle, the state its halo copies need for the force
 * loop ("densities and friends"): state_out [k][5] = {h, A = P/(Omega rho^2),
 * rho, c, Balsara f}. */
int sph_export_state(sph_ctx* ctx, int64_t k, const int32_t* idx, float* state_out);

/* Before sph_force: the halo particles' state [n_halo][5] (same layout, halo order). */
int sph_import_halo_state(sph_ctx* ctx, const float* state);

/* ---- NCCL transport of the slab ring. NCCL is loaded at run time
 * (libnccl.so.2); SPH_E_NCCL if it is missing or a call fails. Rank r's neighbours are
 * lower = r-1 and upper = r+1 (mod cfg.nranks). All buffers are device memory, enqueued on
 * the context's stream (synchronised before return under SPH_F_SYNC); every rank of the
 * communicator must make the same calls in the same order. */

/* Rank 0: a new NCCL unique id (128 bytes) for sph_comm_init; broadcast it to the other ranks
 * with any host transport (e.g. torch.distributed). */
int sph_comm_unique_id(uint8_t* id_out);

/* ncclCommInitRank(cfg.nranks, id, cfg.rank) on the context's device; collective. */
int sph_comm_init(sph_ctx* ctx, const uint8_t* id);

/* The counts of the next exchange: this rank sends n_lo rows to its lower and n_hi rows to
 * its upper neighbour; returns the rows it will receive from each (host values). */
int sph_halo_counts(sph_ctx* ctx, int64_t n_lo, int64_t n_hi, int64_t* m_lo, int64_t* m_hi);

/* Ring exchange of fp32 rows of `cols` values: send_lo [n_lo][cols] -> lower neighbour,
 * send_hi [n_hi][cols] -> upper neighbour; recv_lo [m_lo][cols] <- lower neighbour's send_hi,
 * recv_hi [m_hi][cols] <- upper neighbour's send_lo (counts from sph_halo_counts). Used for
 * the two halo exchanges of an evaluation: x, v, m, u, h0 of the sph_halo_select particles
 * before sph_build_cells_halo, and the sph_export_state rows before sph_import_halo_state. */
int sph_halo_exchange(sph_ctx* ctx, int32_t cols, const float* send_lo, int64_t n_lo, const float* send_hi,
                      int64_t n_hi, float* recv_lo, int64_t m_lo, float* recv_hi, int64_t m_hi);

/* In-place all-reduce of a device buffer over the communicator: dtype 0 = fp64, 1 = int64;
 * op 0 = sum, 1 = max (slab-cut histograms, the global max h for the halo width). */
int sph_allreduce(sph_ctx* ctx, void* buf, int64_t count, int32_t dtype, int32_t op);

/* Work-weighted histogram (NEXT-f3, work-weighted partition; the paper weights its cell
 * graph by the cost of the pair tasks): hist_out[b] = sum of w[i] (int32 work
 * units, negative counted as 0) over the particles with x in bin b of [lo, hi). Integer
 * sums, so the cuts taken from it are reproducible. */
int sph_x_histogram_weighted(sph_ctx* ctx, int64_t n, const float* x, const int32_t* w, double lo, double hi,
                             int32_t nbins, int64_t* hist_out);

/* Particles that left the slab [lo, hi) (re-partition / drift): idx_lo_out = ascending
 * indices with x < lo (to the lower neighbour), idx_hi_out = those with x >= hi (to the
 * upper one); each has room for n entries, counts_out[0..1] their lengths. */
int sph_slab_leavers(sph_ctx* ctx, int64_t n, const float* x, double lo, double hi, int32_t* idx_lo_out,
                     int32_t* idx_hi_out, int64_t* counts_out);

/* The halo width the last sph_density call on a context with a halo needs: the largest h of
 * an owned particle lying within h of a slab face (every partner of an owned particle, and
 * every foreign particle whose h reaches one, then lies within that distance of the face).
 * Set also when the call returned SPH_E_NOCONV because it exceeded cfg.halo_width: the caller
 * sends the missing band [width, h_max) of its faces and evaluates again (slab.py). */
int sph_halo_required(sph_ctx* ctx, double* h_max);

/* ---- CUDA IPC for the peer-store halo (NEXT-f3: the pack kernel of one rank writes its rows
 * straight into the neighbour's receive buffer over NVLink, P:1107-1146's communication
 * without a separate send; slab.py PeerTransport). Handles are 64 opaque bytes the caller
 * hands to the other process with any host transport. Everything created or opened here is
 * released by sph_destroy. */

/* A device buffer of `bytes` other processes can open (cudaMalloc'd on its own); *dev_ptr
 * is its address here, handle[64] its IPC handle. */
int sph_ipc_alloc(sph_ctx* ctx, int64_t bytes, void** dev_ptr, uint8_t* handle);
/* Map another process's sph_ipc_alloc buffer (peer access enabled lazily): *dev_ptr. Device
 * kernels of this context (sph_halo_pack, sph_export_state) may then write into it. */
int sph_ipc_open(sph_ctx* ctx, const uint8_t* handle, void** dev_ptr);
/* An interprocess event (no timing): *id for record / wait, handle[64] for the other side. */
int sph_ipc_event_create(sph_ctx* ctx, int32_t* id, uint8_t* handle);
/* Open another process's event: *id. */
int sph_ipc_event_open(sph_ctx* ctx, const uint8_t* handle, int32_t* id);
/* Record event id on the context's stream / make the stream wait for its last record (the
 * caller orders record before wait across processes, e.g. by a host message sent after the
 * record). */
int sph_ipc_event_record(sph_ctx* ctx, int32_t id);
int sph_ipc_event_wait(sph_ctx* ctx, int32_t id);

/* Replace cfg.halo_width (after the band of a wider halo was received). width >= 0. */
int sph_set_halo_width(sph_ctx* ctx, double width);

/* Histogram of x over [lo, hi) into nbins bins (for count-quantile slab cuts). */
int sph_x_histogram(sph_ctx* ctx, int64_t n, const float* x, double lo, double hi, int32_t nbins,
                    int64_t* hist_out);

/* Pseudo-Verlet reuse of the cells: new positions x [n][3] and smoothing
 * lengths h0 [n] (> 0) of the particles of the last sph_build_cells (same n, no halo). When
 * no particle moved by more than a tenth of the smallest h0 since that build (and no leaf
 * is presorted), the sort, the hierarchy and the target groups are kept and every node
 * test is widened by the drift; otherwise this is sph_build_cells(x, h0). Then the
 * neighbour lists as in sph_build_cells. stats.cells_reused (sph_density) tells which. */
int sph_update_cells(sph_ctx* ctx, const float* x, const float* h0);

/* ---- active subset (the paper's multiple time-stepping: only active
 * particles are "included in the density and force calculations"). active [n] (caller
 * order, device or host; copied), 1 = target, 0 = source only; NULL clears it (all
 * active). Applies from the next sph_build_cells, which must then get h0 (the inactive
 * particles' current h). Inactive particles keep their h, their sph_density state (the
 * A, rho, c, f of their last evaluation, used as sources by sph_force) and their output
 * entries: with a mask, outputs must be device arrays (SPH_E_ARG otherwise). */
int sph_set_active(sph_ctx* ctx, int64_t n, const uint8_t* active);

/* ---- the step around the hot path (first part). Device arrays in the
 * caller's order; enqueued on the context's stream (synchronised under SPH_F_SYNC).
 * Velocity-Verlet: kick(dt/2), drift(dt), build + density + force, kick(dt/2). */

/* v[n][3] += a[n][3] dt; u[n] += dudt[n] dt (u and dudt may both be NULL). */
int sph_kick(sph_ctx* ctx, int64_t n, float* v, float* u, const float* a, const float* dudt, float dt);

/* Individual time steps: v[n][3] += a[n][3] dt[i], u[n] += dudt[n] dt[i] with
 * dt [n] (device); dt[i] = 0 leaves particle i unchanged. */
int sph_kick_each(sph_ctx* ctx, int64_t n, float* v, float* u, const float* a, const float* dudt, const float* dt);

/* Time-step limiter support: after sph_force, for every target i of that call and every j
 * with r_ij < max(h_i, h_j), out[j] = min(out[j], val[i]). val, out [n] caller order,
 * device, positive values (out is read and updated). Deterministic (min). */
int sph_neighbour_min(sph_ctx* ctx, const float* val, float* out);

/* Individual power-of-two time steps, the bin arithmetic of a multiple
 * time-stepping integrator, in integer ticks of dt_min. For every particle with active[i] != 0
 * (all if active is NULL): ticks_out[i] = the largest power of two s <= min(dt_i / dt_min,
 * 2^n_bins) (dt_i of Eq. 6 from h and vsig, c_cfl) that divides ti (a new step starts on its
 * own grid), and with cap2 != 0 at most 2 ticks_in[i] (a step grows at most 2x at a time);
 * inactive particles keep ticks_in[i] (ticks_in is required when active is given). All arrays
 * device memory; ticks int64. */
int sph_timebins(sph_ctx* ctx, int64_t n, const float* h, const float* vsig, float c_cfl, double dt_min,
                 int32_t n_bins, int64_t ti, const uint8_t* active, const int64_t* ticks_in, int32_t cap2,
                 int64_t* ticks_out);

/* Time-step limiter wake-up: an inactive particle whose step exceeds 4 lim[i] ticks (lim: the
 * smallest new step of a force neighbour, from sph_neighbour_min) ends its step at the next
 * point of the grid of the largest power of two <= 4 lim[i] after ti_end, never later than its
 * current end ti_begin[i] + ticks[i]. ticks[i] is shortened in place; kick[i] = (new - old)
 * ticks x dt_min / 2 (the correction of its opening half kick), else 0. Device arrays. */
int sph_timebins_wake(sph_ctx* ctx, int64_t n, const uint8_t* active, const float* lim, int64_t ti_end,
                      const int64_t* ti_begin, int64_t* ticks, double dt_min, float* kick);

/* x[n][3] += v[n][3] dt, wrapped back into [0, L) per axis (requires |v dt| < L). */
int sph_drift(sph_ctx* ctx, int64_t n, float* x, const float* v, float dt);

/* Eq. 6: dt_i = c_cfl 2 h_i / vsig_i with vsig_i = max_j (c_i + c_j
 * + max{0, -3 r_ij . v_ij / r_ij}) from sph_force's vsig_out (+inf where vsig = 0).
 * dt_out [n] (device, or NULL); *dt_min_out (host) = min_i dt_i. The paper uses c_cfl = 1/4
 * (P:1353). */
int sph_timestep(sph_ctx* ctx, int64_t n, const float* h, const float* vsig, float c_cfl, float* dt_out,
                 float* dt_min_out);

/* ---- structure introspection (tests and tools; not on the hot path). Copies one of the
 * context's internal arrays to the HOST buffer `out` (room for `cap` elements) and sets
 * *count to its element count (nothing is copied when cap < count). `what`:
 *   SPH_X_PERM     uint32 [n]        cell order -> caller index (the sort's permutation)
 *   SPH_X_GROUPS   int32 [ng][4]     target groups {node, first, count, 0} (cell order)
 *   SPH_X_LIST_OFF int64 [ng]        interaction-list offset of each group
 *   SPH_X_LIST_LEN int32 [ng]        interaction-list length of each group
 *   SPH_X_LIST     uint32 [entries]  interaction-list entries (image code << 27) | source
 *   SPH_X_NODES    int32 [nodes][4]  {first, count, first child or -1, octant mask | level << 8}
 *   SPH_X_SORTOFF  int64 [nodes]     offset of a node's 13 presorted lists, -1 if none
 *   SPH_X_SORTED   {float key, int32 idx} [entries]  presorted lists, 13 per node
 *   SPH_X_XH       float [n][4]      cell-order positions and current h
 * Errors: SPH_E_ARG (unknown `what`, count or out NULL), SPH_E_STATE (no build yet). */
#define SPH_X_PERM 0
#define SPH_X_GROUPS 1
#define SPH_X_LIST_OFF 2
#define SPH_X_LIST_LEN 3
#define SPH_X_LIST 4
#define SPH_X_NODES 5
#define SPH_X_SORTOFF 6
#define SPH_X_SORTED 7
#define SPH_X_XH 8
int sph_debug_export(sph_ctx* ctx, int32_t what, void* out, int64_t cap, int64_t* count);

/* ---- the paper's cell-pair loops, for the sorted-vs-naive ablation (not
 * the hot path). After sph_density: a uniform periodic grid of edge >= max h, each
 * cell with itself and its 13 forward neighbours, the density sums of Eq. 2 by the naive
 * double loop (sorted = 0) or the sorted sweeps with early exit (sorted = 1,
 * P:644-669 with R6/R7, 13 presorted directions per cell). rho_out [n] (caller order, device or
 * host, or NULL) gets rho = (8/pi) h^-3 sum m f at the context's h. counts_out (host, 16 int64):
 * [0] distance tests, [1] directed contributions found, [2..4] particle pairs n_A n_B of face /
 * edge / corner cell pairs, [5..7] their sweep-1 window passes (naive: all pairs), [8..10] their
 * sweep-1 pairs within h_i, [11] cells per axis (x), [12] pair-loop kernel time in ns, [13]
 * presort time in ns. Errors: SPH_E_STATE (no sph_density yet), SPH_E_ARG. */
int sph_pair_ablation(sph_ctx* ctx, int32_t sorted, float* rho_out, int64_t* counts_out);

/* Number of CUDA kernel launches libsph issued on this context since creation
 * (evidence for the bench's gpu_launches). */
int64_t sph_kernel_launches(const sph_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SPH_H */
