/*
 * pi.h -- C ABI of libpi, a B200-native (sm_100a) implementation of the hot path of
 * arXiv 2406.16091 "cutoff-limited pairwise particle interactions on a cell grid with
 * few particles per cell".
 *
 * Citations: "PAPER.md:L" is line L of the paper's LaTeX source (the paper itself, not
 * shipped here); section / algorithm / equation named alongside.
 *
 * What the library computes (§2): for every particle i, the interactions
 * with all j != i such that r_ij < r_c through a kernel K(r_ij); the grid of cells of
 * width >= r_c (§3) only restricts the candidates to the 27 neighbour cells
 * (§5.1).  The pipeline (§2):
 *   a1 cell index of every particle from its position             -> pi_bin
 *   a2 per-cell counts with atomics                               -> pi_bin
 *   a3 prefix sum of the counts (+ M_C, §5.1)       -> pi_bin
 *   a4 out-of-place move into cell-sorted "secondary" arrays      -> pi_bin
 *   a5 launch configuration (sub-box / pencil sizing)             -> pi_interact
 *   a6 interactions with the same and neighbouring cells          -> pi_interact
 *   a7 position update ("their positions are updated", :65)       -> pi_step
 *   a8 X-slab ghost / migration exchange (north star, nranks > 1) -> pi_bin / pi_step
 *
 * Conventions
 *   Pointers: every particle/cell array argument is a CUDA DEVICE pointer owned by the
 *     caller, unless the function name ends in _host (pinned or pageable host memory).
 *     Float arrays must be 16-byte aligned (vectorised loads); NULL is allowed only where
 *     stated.
 *   Ownership: libpi never allocates device memory.  All of its state lives in the
 *     caller-provided workspace (pi_workspace_bytes); pi_create only carves it up.
 *     pi_bin copies its inputs (out of place) and never writes them.
 *   Asynchrony: calls enqueue on cfg.stream and return without synchronising, except
 *     pi_create (NCCL bootstrap when nranks > 1), pi_get_stats and the *_host calls.
 *     pi_bin / pi_interact / pi_step perform no allocation and no host synchronisation,
 *     so they can be captured in a CUDA graph.
 *   Errors: status codes, nothing is thrown across the ABI; pi_last_error() gives text.
 *     Errors detected on the device (particle outside the box, NaN position, capacity
 *     overflow) set a sticky flag reported by the next pi_get_stats (PI_EDEVICE).
 *   Threading: one context per (process, GPU); a context is not thread safe.
 */
#ifndef PI_H_
#define PI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PI_ABI_VERSION 1

#if defined(__GNUC__)
#define PI_API __attribute__((visibility("default")))
#else
#define PI_API
#endif

typedef struct pi_ctx_s *pi_ctx;

typedef enum {
  PI_OK = 0,
  PI_EINVAL = 1,         /* bad argument (see each call)                                  */
  PI_ECAPACITY = 2,      /* n (or arrivals) exceed cfg.capacity                           */
  PI_EINAPPLICABLE = 3,  /* strategy cannot run (PAPER.md:276 sub-box < 27 cells, :354)   */
  PI_ECUDA = 4,          /* CUDA runtime error (text in pi_last_error)                     */
  PI_ENCCL = 5,          /* NCCL error                                                     */
  PI_ESTATE = 6,         /* call out of order (e.g. pi_interact before pi_bin)             */
  PI_EDEVICE = 7         /* sticky device-side error flag was set (see pi_stats.flags)     */
} pi_status;

/* Interaction kernel K(r).  PAPER.md:51-52 (§2) names "the Gaussian function"; the paper's
 * measured kernel is Lennard-Jones (Eq. 1), listed as next work.
 *   PI_K_GAUSSIAN : K(r) = exp(-r^2 / (2 sigma^2)), sigma = kparam[0] (0 -> r_c / 3);
 *                   phi_i = sum_j q_j K(r_ij),  F_i = (q_i / sigma^2) sum_j q_j K(r_ij) (x_i - x_j)
 *                   (F_i = -grad_i of q_i sum_j q_j K).
 *   PI_K_INDICATOR: phi_i = sum_{j: r_ij < r_c} q_j, F = 0        (test kernel: exact counts)
 *   PI_K_CANDIDATE: phi_i = sum_{j in 27 cells, j != i} q_j, F = 0 (test kernel: no cutoff)
 *   PI_K_LJ       : the paper's measured kernel, Eq. (1) as printed with the
 *                   softening of :582 (reading R19): d~ = sqrt(r_ij^2 + eps^2), u = d~ / r,
 *                   K = 4 E0 (u^12 - u^6); phi_i = sum_j q_j K, F_i = -grad_i (q_i sum_j q_j K);
 *                   the cutoff test uses the unsoftened r_ij.  kparam[0] = r (0 -> r_c),
 *                   kparam[1] = eps (>= 0), kparam[2] = E0 (0 -> 1).
 * The two fake kernels of the paper's kernel-cost experiment (Fig. "diffflops", PAPER.md:785-788;
 * reading R22 of DESIGN.md), with the same cutoff test r_ij < r_c:
 *   PI_K_LOWFLOP  : "summing the positions" (5 FLOP per interaction): phi_i = sum_j (x_j + y_j +
 *                   z_j), F_i = sum_j (x_j, y_j, z_j); q is not used.
 *   PI_K_HIGHFLOP : "the Lennard-Jones kernel with 150 added FLOP" (168 FLOP): PI_K_LJ, whose
 *                   potential term u = (d~/r)^12 - (d~/r)^6 goes through 75 FMAs t <- t a + b,
 *                   a = 1 - 2^-7, b = 2^-10 (the affine map A u + B, A = a^75,
 *                   B = b (1 - A) / (1 - a)) before phi_i = sum_j q_j 4 E0 t; F_i as PI_K_LJ;
 *                   kparam as PI_K_LJ.                                                       */
typedef enum {
  PI_K_GAUSSIAN = 0,
  PI_K_INDICATOR = 1,
  PI_K_CANDIDATE = 2,
  PI_K_LJ = 3,
  PI_K_LOWFLOP = 4,
  PI_K_HIGHFLOP = 5
} pi_kernel;

/* Interaction strategy (a6).
 *   PI_A_GLOBAL  : Par-Part-NoLoop (Alg. 1, §4.1): one thread per target,
 *                  sources read from global memory through L1/L2.  The paper's baseline.
 *   PI_A_FULLLOAD: All-in-SM / full load (Alg. 4, §5.1): a 3-D sub-box
 *                  plus its ghost shell staged in shared memory (cp.async.bulk), local
 *                  offsets from the global prefix array.
 *   PI_A_XPENCIL : X-pencil (Alg. 5, §5.2), re-designed to stream the
 *                  9 neighbour pencils of a target pencil along X through shared memory.
 *   PI_A_AUTO    : the fastest measured strategy for the workload: the global-memory kernel
 *                  below 3 particles per cell (mean), the X-pencil above.
 *   PI_A_XPREG   : X-pencil-reg (§5.3): the targets
 *                  of a sub-box of cells in registers, the (By+2)(Bz+2) source X-pencils around
 *                  it staged one after the other, the box's own records copied to shared memory
 *                  from the registers.  Needs the sorted records (pi_bin / pi_step write them).
 *   PI_A_HALF    : Newton-3rd-law half-shell: every unordered pair
 *                  evaluated once, by the target whose upper half-neighbourhood holds the
 *                  source (4 of the 8 neighbour rows, the rest of its own row after it), and
 *                  credited to both (phi_j gets q_i K, F_j = -F_i: Eq. (1));
 *                  the source's share is a vector reduction into the sorted-order output.
 *                  One thread per target as PI_A_GLOBAL; needs the sorted records.  */
typedef enum {
  PI_A_GLOBAL = 0,
  PI_A_FULLLOAD = 1,
  PI_A_XPENCIL = 2,
  PI_A_AUTO = 3,
  PI_A_XPREG = 4,
  PI_A_HALF = 5
} pi_algo;

typedef struct {
  /* Global grid (PAPER.md:54-56 §2, :93 §3).  Cells are cubes of width cell_width; the box
   * is [origin, origin + dims * cell_width); linear cell index is X-fastest,
   * lin = cx + dims[0] * (cy + dims[1] * cz).  Boundaries are open.      */
  float origin[3];
  float cell_width;          /* must be >= r_c; > 0                          */
  int32_t dims[3];           /* each >= 1; dims[0] divisible by nranks                      */
  float r_c;                 /* cutoff radius, > 0                                           */
  int32_t kernel;            /* pi_kernel                                                    */
  float kparam[4];           /* kernel parameters: Gaussian kparam[0] = sigma (0 -> r_c/3);
                                LJ kparam[0..2] = r, eps, E0 (see pi_kernel)                  */
  int64_t capacity;          /* max particles resident on this rank (owned + ghosts)        */
  void *stream;              /* cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)  */
  int32_t rank, nranks;      /* X-slab decomposition (north star); nranks >= 1               */
  const void *nccl_unique_id;/* 128-byte ncclUniqueId shared by all ranks (pi_nccl_unique_id
                                on one rank, broadcast by the caller); NULL iff nranks == 1.
                                Testing: "PILOCAL:<key>" links the nranks contexts of ONE
                                process (one host thread per context) without NCCL.          */
  int32_t x_subcells;        /* internal X resolution of the binning: inside each cell the
                                particles are ordered by sub-cell floor(sx (t - c)), t the
                                contract's scaled coordinate (R18), so the X-pencil
                                can skip sources farther than r_c along X; 1, 2, 4, 8 or 16
                                (0 -> 4: configs[4] step 19.9 -> 19.4 ms against 2, r02).
                                Counts, offsets and M_C stay per cell.                       */
  int32_t reserved[7];       /* must be zero                                                 */
} pi_config;

typedef struct {
  int64_t n_owned;           /* particles owned by this rank after the last pi_bin/pi_step  */
  int64_t n_ghost;           /* ghost (source-only) particles staged from neighbour ranks   */
  int32_t max_per_cell;      /* M_C of the last binning                       */
  int32_t flags;             /* sticky device error bits: 1 out-of-box/NaN position,
                                2 capacity overflow (particles or a8 messages), 4 internal
                                (e.g. a particle moved more than one slab in one step),
                                8 a pi_bin particle outside this rank's slab                 */
  int64_t candidates;        /* ordered candidate pairs of the last interaction (C)          */
  int64_t fallback_cells;    /* target cells the staged kernels could not stage: computed by
                                the Par-Cell-SM pass (X-pencil: cells whose window alone
                                exceeds a slot; full load: the cells of boxes that do not fit) */
  int64_t migrants_in;       /* particles received by the last migration (nranks > 1)       */
  int64_t migrants_out;      /* particles sent by the last migration (nranks > 1)           */
  int64_t steps;             /* pi_step calls so far                                          */
  int64_t exchange_bytes;    /* a8: payload bytes this rank sent to its neighbours so far      */
  double phase_ms[4];        /* device time of the last bin (a1-a4), interaction (a5-a7),
                                exchange (a8) and host-path copies, from CUDA events recorded
                                on the context stream around each phase (the overlapped
                                exchange: on the library's exchange stream)                   */
  int64_t overlapped_steps;  /* a8: pi_step calls whose exchange ran beside the interior
                                interaction (pi_tuning.exchange_overlap)                      */
  int64_t reserved[2];
} pi_stats;

/* Tuning knobs of the launch configuration (a5).  Zero fields mean "library default".   */
typedef struct {
  int32_t xpencil_len;       /* X-pencil: target cells per work item (row segment); default
                                from the mean density: 64 at >= 8 per cell, 128 at >= 4,
                                256 below                                                   */
  int32_t xpencil_cap;       /* X-pencil: records one staging slot holds (default: as many as
                                the shared memory of the block's slots allows); a segment
                                that does not fit is split into rounds, a cell whose window
                                alone does not fit is listed for the Par-Cell-SM pass       */
  int32_t fullload_box[3];   /* full load: target sub-box (interior) dims (8, 4, 4)         */
  int32_t fullload_cap;      /* full load: staged particles per block                       */
  int32_t threads;           /* threads per block of the staged kernels                     */
  int32_t xpencil_slots;     /* X-pencil: staging slots per block (2..4; default 2)         */
  int32_t xpencil_targets;   /* X-pencil: targets per consumer lane, 1 or 2 (default 1; 2
                                reads each staged source once for two consecutive targets;
                                the CANDIDATE test kernel always walks one); 3 = cell groups:
                                a warp per target cell, 32 / n lanes per target over the
                                union window of the cell (measured slower)     */
  int32_t exchange_full;     /* a8 (nranks > 1): 0 (default) = two-phase exchange, the counts
                                first, then exactly the counted records (one stream
                                synchronisation per exchange); 1 = the whole fixed-capacity
                                messages, no host synchronisation (CUDA-graph capturable)     */
  int32_t xpencil_layout;    /* X-pencil staging: 0 (default) = the 9 pencils back to back (9
                                runs per target; xpencil_targets applies); 1 = X-sub-cell-
                                interleaved (a target's candidates are one contiguous range,
                                one thread per target pair; measured slower)     */
  int32_t exchange_overlap;  /* a8 (nranks > 1, X-pencil, >= 4 owned X layers): 0 (default) =
                                the step computes the first and last 2 owned layers first, then
                                the interior while a second (library-created) stream exchanges
                                the migrants and the next step's ghosts; 1 = serial exchange at
                                the start of the next step                                    */
  int32_t reserved[3];
} pi_tuning;

PI_API int32_t pi_abi_version(void);

/* a8 X-slab decomposition (north star; the paper is single-GPU).  Rank r of P = nranks owns
 * the global X cells [r Lx, (r+1) Lx), Lx = dims[0] / P, all Y and Z.  Its local grid has
 * Lx + 2 X layers: local 0 and Lx + 1 are ghost layers (source-only copies of the
 * neighbours' boundary layers), local 1..Lx are owned; local X = global X - gx_off.
 * out[0] Lx, out[1] first owned global X cell, out[2] one past the last, out[3] local X
 * layers, out[4] gx_off, out[5] own_lo, out[6] own_hi (local, half-open), out[7] record
 * capacity of each a8 message.  Host only, no context needed.  Errors: PI_EINVAL.       */
PI_API pi_status pi_slab_info(const pi_config *cfg, int64_t out[8]);

/* 128-byte ncclUniqueId from the NCCL library libpi uses (libnccl.so.2, dlopen'ed).
 * Errors: PI_EINVAL (NULL), PI_ENCCL (library missing).                                    */
PI_API pi_status pi_nccl_unique_id(void *out128);

/* Bytes of device workspace a context with this configuration needs (0 on bad config).   */
PI_API size_t pi_workspace_bytes(const pi_config *cfg);

/* Create a context inside `workspace` (device memory, >= pi_workspace_bytes, 256-B
 * aligned).  With nranks > 1 this is collective over the ranks (NCCL communicator
 * bootstrap from cfg->nccl_unique_id) and synchronises.
 * Errors: PI_EINVAL (cell_width < r_c, dims <= 0, dims[0] % nranks, r_c <= 0, workspace
 * too small or misaligned, NULL out), PI_ENCCL, PI_ECUDA.                                  */
PI_API pi_status pi_create(const pi_config *cfg, void *workspace, size_t ws_bytes, pi_ctx *out);
PI_API pi_status pi_destroy(pi_ctx ctx);
PI_API pi_status pi_set_stream(pi_ctx ctx, void *stream);
PI_API pi_status pi_set_tuning(pi_ctx ctx, const pi_tuning *t);

/* a1-a4 (+a8 when nranks > 1): bin n particles (SoA, device pointers, §2) into
 * the context's cell-sorted state.  id may be NULL (ids default to 0..n-1).  Positions must
 * lie in the box; a particle on the upper face clamps into the last cell.  nranks > 1: the
 * call is collective, each rank passes the particles of ITS slab (pi_slab_info; others
 * raise flag 8) and the first / last owned X layers are exchanged as ghosts before the
 * owned + ghost particles are binned together.  Errors: PI_EINVAL (n < 0, NULL or
 * misaligned pointer with n > 0), PI_ECAPACITY (n > capacity), PI_ENCCL.                   */
PI_API pi_status pi_bin(pi_ctx ctx, int64_t n, const float *x, const float *y, const float *z, const float *q,
                 const int32_t *id);

/* a5-a6: interactions of every binned particle with its candidates (same and 26
 * neighbouring cells, j != i, r_ij < r_c).  Outputs are written in the caller order of the
 * last pi_bin (length n); any output pointer may be NULL (results stay in the context's
 * sorted state, see pi_get_particles).  Errors: PI_ESTATE (no binning yet, or the sorted
 * state came from pi_step and caller-order outputs were requested), PI_EINAPPLICABLE.      */
PI_API pi_status pi_interact(pi_ctx ctx, pi_algo algo, float *phi, float *fx, float *fy, float *fz);

/* One time step: bin the current positions, interact, then x <- x + dt F with reflecting
 * walls (reading of PAPER.md:65), in sorted order.  Collective when
 * nranks > 1: before re-binning, owned particles whose updated global X cell left the slab
 * migrate to rank -1 / +1 (at most one slab per step, else flag 4), then the ghost layers
 * are exchanged again.  The first call after pi_bin reuses that binning.  With the X-pencil
 * and >= 4 owned X layers (pi_tuning.exchange_overlap = 0) the exchange is overlapped: the
 * step computes the first and last 2 owned layers first, then the interior while the
 * migrants and the next step's ghosts are exchanged on a second stream; the call returns
 * with the context stream ordered after that exchange.  The overlap needs |dt F| < w per
 * step (else flag 4, as for migration beyond one slab).                                     */
PI_API pi_status pi_step(pi_ctx ctx, pi_algo algo, float dt);

/* End-to-end call on HOST buffers: copies x,y,z,q (n floats each) host->device, bins,
 * interacts and copies phi,fx,fy,fz device->host, then synchronises the stream.  Host
 * buffers should be pinned for full bandwidth.  Outputs in input order; NULL allowed.      */
PI_API pi_status pi_run_host(pi_ctx ctx, pi_algo algo, int64_t n, const float *x, const float *y, const float *z,
                      const float *q, float *phi, float *fx, float *fy, float *fz);

/* Pipelined end-to-end runs on HOST buffers, for a stream of independent inputs (one rank):
 * pi_run_host_submit enqueues what pi_run_host does -- H2D x,y,z,q, bin, interact, D2H
 * phi,F -- and returns without synchronising; up to three runs are in flight (a fourth submit
 * first waits for the oldest), each on its own third of the workspace's I/O buffers, with the
 * host->device copies on one internal stream, the kernels on the context stream and the
 * device->host copies on another, so run k+1's upload and run k-1's download overlap run k's
 * kernels (PCIe is full duplex).  The caller keeps every host buffer of a run valid and
 * unread until pi_run_host_wait, which blocks until all submitted runs' outputs are in host
 * memory (and orders the context stream after them).  Same arguments and errors as
 * pi_run_host; the introspection calls see the state of the latest submitted run.         */
PI_API pi_status pi_run_host_submit(pi_ctx ctx, pi_algo algo, int64_t n, const float *x, const float *y,
                                    const float *z, const float *q, float *phi, float *fx, float *fy, float *fz);
PI_API pi_status pi_run_host_wait(pi_ctx ctx);

/* Introspection (device pointers, async, any may be NULL):
 *   cell_of[n]  cell index of each particle of the last pi_bin, caller order   (a1)
 *   counts[Nc]  particles per cell (local grid when nranks > 1)                (a2)
 *   offsets[Nc+1] exclusive prefix, offsets[Nc] = n                            (a3)
 *   perm[n]     sorted slot -> caller index of the last pi_bin                  (a4)
 * nranks > 1: cells are LOCAL (Nc = (Lx + 2) dims[1] dims[2], see pi_slab_info), the sorted
 * state holds n_owned + n_ghost slots, perm is -1 on ghost slots and offsets[Nc] =
 * n_owned + n_ghost.                                                                          */
PI_API pi_status pi_get_binning(pi_ctx ctx, int32_t *cell_of, int32_t *counts, int32_t *offsets, int32_t *perm);

/* Sorted state (device pointers, async, any may be NULL): positions, values, ids and the
 * last interaction's outputs of the n_owned owned particles, in cell-sorted order (after
 * pi_step: the updated positions, not yet re-binned).  nranks > 1: the owned particles
 * only (ghosts skipped, migrants of the next step still included), order unspecified;
 * arrays must hold pi_stats.n_owned entries.                                                */
PI_API pi_status pi_get_particles(pi_ctx ctx, float *x, float *y, float *z, float *q, int32_t *id, float *phi,
                           float *fx, float *fy, float *fz);

/* Synchronises the stream and fills *out.  Returns PI_EDEVICE if a sticky flag is set.      */
PI_API pi_status pi_get_stats(pi_ctx ctx, pi_stats *out);

/* P, the statistic of SURVEY.md §5 beside C: the ordered pairs (i, j), j != i, with r_ij < r_c
 * (strict) over this rank's owned targets in the current sorted state (the state
 * the last interaction used), counted by a separate pass with the global baseline's walk and
 * fp32 arithmetic -- the interaction kernels do not count it (it would cost the hot loop).
 * *pairs: host int64.  Synchronises.  Errors: PI_EINVAL (NULL), PI_ESTATE (before pi_bin).    */
PI_API pi_status pi_count_pairs(pi_ctx ctx, int64_t *pairs);

PI_API const char *pi_last_error(pi_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* PI_H_ */
