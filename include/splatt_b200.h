/*
 * splatt_b200.h — C ABI of the B200-native sparse CP-ALS hot path.
 *
 * The method: CP-ALS (Algorithm 1) over CSF-compressed sparse
 * tensors, whose dominant step is the per-mode MTTKRP
 * M_n = X_(n) (KRP_{m != n} A_m)  (lines 5/8/11).
 * The calls follow the problem statement of BASELINE.json's north star:
 *   splatt_csf_build(coo, nmodes, dims), splatt_mttkrp(csf, mode, factors, out),
 *   splatt_cpd_als(coo, rank, max_iters, tol, seed) -> factors, lambda, fit.
 * Readings of passages the paper leaves open are listed in DESIGN.md §2.
 *
 * Conventions (every call):
 *  - Every function returns splatt_status (0 = OK) unless noted.  On error the
 *    context keeps a message (splatt_last_error).  No call throws or aborts.
 *  - Argument errors are detected synchronously, before any device work.
 *  - Indices are 0-based uint32; values and factors are fp64.
 *  - Factor / output matrices are row-major I_n x R with a leading dimension ld
 *    (elements between consecutive rows), ld >= R.
 *  - Ownership: the caller owns every pointer it passes (COO arrays, factors,
 *    outputs); the library never frees caller memory.  The library owns
 *    splatt_ctx (free with splatt_ctx_destroy) and splatt_csf (splatt_csf_free).
 *  - Memory spaces: splatt_csf_build and splatt_cpd_als accept host OR device
 *    pointers for the COO and the outputs (detected with cudaPointerGetAttributes;
 *    host buffers are copied inside the call).  splatt_mttkrp takes device
 *    pointers only.
 *  - Streams: every device operation is ordered on the context stream (the one
 *    passed to splatt_ctx_create, else the library's own).  splatt_csf_build and
 *    splatt_mttkrp return after enqueueing (asynchronous faults surface as
 *    SPLATT_ERR_CUDA from a later call or splatt_ctx_sync); splatt_cpd_als
 *    returns when its outputs are written.
 *  - Threading: one context per host thread; distinct contexts are independent.
 *  - No CPU fallback exists: every arithmetic step runs in the library's CUDA
 *    kernels on the context's device.
 */
#ifndef SPLATT_B200_H
#define SPLATT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPLATT_OK = 0,
  SPLATT_ERR_BADINPUT = -1,    /* invalid argument (see each call)                       */
  SPLATT_ERR_NOMEM = -2,       /* device or host allocation failed                      */
  SPLATT_ERR_SINGULAR = -3,    /* Cholesky of V failed after the ridge retry (C-7)      */
  SPLATT_ERR_CUDA = -4,        /* CUDA runtime error (message in splatt_last_error)     */
  SPLATT_ERR_NCCL = -5,        /* NCCL error or NCCL library not loadable               */
  SPLATT_ERR_EMPTY = -6,       /* ||X|| = 0: the fit is undefined         */
  SPLATT_ERR_UNSUPPORTED = -7  /* valid but outside this build (nnz >= 2^31)           */
} splatt_status;

enum { SPLATT_MAX_NMODES = 8, SPLATT_MAX_RANK = 128 };

/* CSF allocation policy (the lock / no-lock dichotomy of
 * PAPER.md:253-275, 469-470).
 *   ALL: one CSF rooted at every mode, so every MTTKRP is a ROOT ("no-lock") traversal
 *        with owned output rows.  N CSFs of memory.
 *   ONE: one CSF rooted at the shortest mode (ties -> lowest id), the other modes below
 *        it by ascending length; the mode at level l > 0 runs the INTERNAL (l < N-1) or
 *        LEAF (l = N-1) kernel, whose output rows are shared between parents and are
 *        accumulated with asynchronous bulk fp64 reductions at L2 (the hottest rows
 *        privatised per lane group first) — the GPU's replacement of the paper's mutex
 *        pool.
 *   TWO: ONE's CSF plus one rooted at the longest mode (the last in ascending-length
 *        order); both roots run ROOT kernels, every other mode its level in the first.  */
enum { SPLATT_CSF_ALL = 0, SPLATT_CSF_ONE = 1, SPLATT_CSF_TWO = 2 };

typedef struct splatt_ctx splatt_ctx;   /* device, stream, allocator pool, optional comm */
typedef struct splatt_csf splatt_csf;   /* device-resident CSF set (trees immutable; MTTKRP
                                           scratch built lazily, see splatt_mttkrp)      */
typedef struct splatt_loopback splatt_loopback; /* in-process group of logical ranks     */

/* Sparse tensor in coordinate form (SoA).  nmodes in [3, 8]; nnz >= 1;
 * dims[m] in [1, 2^32); ind[m][p] < dims[m]; duplicates are kept as distinct
 * adjacent leaves in input order.                                 */
typedef struct {
  int32_t         nmodes;
  uint64_t        nnz;
  uint64_t        dims[SPLATT_MAX_NMODES];
  const uint32_t* ind[SPLATT_MAX_NMODES];
  const double*   vals;
} splatt_coo;

/* Caller-allocated CP-ALS outputs (Alg. 1 line 14).                */
typedef struct {
  double*  factors[SPLATT_MAX_NMODES]; /* I_n x R, row-major, ld = R; host or device      */
  double*  lambda;                     /* R weights; host or device                        */
  double   fit;                        /* fit after the last iteration (C-10)              */
  int32_t  iters;                      /* iterations executed                              */
  double*  fit_history;                /* optional (NULL): max_iters doubles, host memory  */
} splatt_kruskal;

/* Per-call measurements, filled by splatt_cpd_als_ex when non-NULL.  Times are
 * seconds from CUDA events on the context stream, summed over the call, in the
 * categories of Table III plus COMM; counters are exact.  The R x R
 * inverse and the fit run on a side stream overlapped with the MTTKRP: their spans
 * (including any wait for a free SM) are reported apart, in t_aux_*.                */
typedef struct {
  double   t_mttkrp;        /* all MTTKRP kernel launches (the output zero-fill before */
                            /*   a ROOT launch is excluded; it is not counted anywhere)  */
  double   t_build;         /* validation + COO->CSF build ("Sort")                     */
  double   t_ata;           /* Hadamard of Grams + Gram refresh ("Mat A^TA")           */
  double   t_norm;          /* partial reduction + lambda ("Mat norm"); one rank: on the  */
                            /*   side stream, overlapped with the next MTTKRP             */
  double   t_fit;           /* fit ("CPD fit")                                          */
  double   t_inverse;       /* Cholesky + row solves ("Inverse")                        */
  double   t_comm;          /* NCCL collectives (0 on one GPU)                          */
  double   t_loop;          /* whole ALS loop (all iterations)                          */
  double   mttkrp_alg_bytes;/* sum over launches of the algorithmic bytes B_alg(n)     */
  uint64_t mttkrp_launches; /* MTTKRP kernel launches                                   */
  uint64_t kernel_launches; /* every library kernel launched by the call                */
  uint64_t csf_nodes[SPLATT_MAX_NMODES][SPLATT_MAX_NMODES]; /* [csf][level] local nodes */
  int32_t  iters;
  int32_t  nranks;
  double   t_call;          /* device time from the call's first to its last stream op   */
  double   t_host_sync;     /* host seconds spent blocked in the call's stream syncs     */
  int32_t  host_syncs;      /* host<->device synchronisations inside the call            */
  double   t_aux_inverse;   /* V^-1 (Hadamard + Gauss-Jordan) spans on the side stream,  */
  double   t_aux_fit;       /*   and fit spans: overlapped with MTTKRP, not in t_inverse  */
  double   mttkrp_min_bytes;/* sum over launches of the compulsory bytes: tree once,      */
                            /*   referenced factor rows once, output once */
  int32_t  exchange;        /* SPLATT_XCHG_* the call's factor-row exchange ran as (0 on   */
                            /*   one rank)                                                  */
} splatt_stats;

/* ---------------------------------------------------------------- context */
/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t to order
 * all work on (e.g. torch.cuda.current_stream().cuda_stream; pass cudaStreamLegacy,
 * i.e. (void*)1, for the legacy default stream), or NULL for a library-owned
 * non-blocking stream.  *out is set only on success.                             */
splatt_status splatt_ctx_create(splatt_ctx** out, int device, void* cuda_stream);
void          splatt_ctx_destroy(splatt_ctx* ctx);
/* Wait for all work on the context stream; reports asynchronous faults.         */
splatt_status splatt_ctx_sync(splatt_ctx* ctx);
/* Last error message of this context ("" if none); valid until the next call.   */
const char*   splatt_last_error(const splatt_ctx* ctx);
const char*   splatt_version(void);

/* ------------------------------------------------- multi-GPU (one process per GPU)
 * every rank passes the same full COO; nonzeros are partitioned by
 * root slices of each mode's CSF (splatt_partition), each rank owns the output rows
 * of its slice range, updated factor rows are all-gathered and the R x R Grams,
 * column maxima and the fit inner product are combined over the ranks with NCCL (one
 * all-gather of the ranks' partials, reduced in rank order on every rank).
 * splatt_comm_unique_id: rank 0 only; writes 128 bytes (ncclUniqueId), to be
 * broadcast by the caller (e.g. torch.distributed).  splatt_ctx_set_comm: collective
 * over the nranks ranks (ncclCommInitRank).  NCCL is loaded at run time
 * (libnccl.so.2); failure -> SPLATT_ERR_NCCL.  id128 = NULL (nranks 1) removes the
 * communicator; nranks = 1 with an id creates a one-rank NCCL communicator, which runs
 * the sharded code path (partition, compaction, collectives) on a single GPU.         */
splatt_status splatt_comm_unique_id(void* id128);
splatt_status splatt_ctx_set_comm(splatt_ctx* ctx, const void* id128, int nranks, int rank);

/* How a sharded context splits each mode's nonzeros:
 *   AUTO (default): per mode, NNZ where the best SLICES cut leaves a rank more than
 *           max(1% of nnz/G, 2^18) nonzeros above the mean (the excess MTTKRP time then
 *           outweighs NNZ's extra small all-reduce), else SLICES.
 *   SLICES (P1): contiguous ranges of whole root slices, the optimal cut of C-14
 *           (splatt_partition); every rank owns the rows of its slices.  Load imbalance is
 *           bounded by the heaviest slice (power-law tensors: up to 14% of nnz in one slice).
 *   NNZ (P2, §8(f) NEXT-2): the mode's nonzeros in slice-major order (slices ascending, a
 *           slice's nonzeros in input order) cut into equal ranges [floor(g nnz/G),
 *           floor((g+1) nnz/G)); a slice may be split.  Its row belongs to the rank holding
 *           its first nonzero; the other ranks' partial rows of the <= G-1 split slices are
 *           summed into it with one all-reduce of (split slices) x ld doubles per mode,
 *           before the solve.  Results differ from SLICES by rounding only.
 * Errors: BADINPUT (unknown mode).                                                       */
enum { SPLATT_PART_SLICES = 0, SPLATT_PART_NNZ = 1, SPLATT_PART_AUTO = 2 };
splatt_status splatt_ctx_set_partition(splatt_ctx* ctx, int32_t mode);

/* How a sharded context shares each mode's solved factor rows (SURVEY.md §8(e) step 5,
 * "updated factor rows are shared"; PAPER.md:212-213, :606 distributed SPLATT):
 *   COLLECTIVE (default): after the row solve, an all-gather of the owned row ranges (NCCL
 *           grouped broadcasts), serialised behind the solve kernel.
 *   PEER:   the row-solve kernel itself stores every solved row at the same offset of every
 *           peer's factor matrix (peer-to-peer stores over NVLink / NVSwitch from inside the
 *           kernel: the transfer overlaps the solve slab by slab and no separate all-gather
 *           runs).  The factor matrices then live in one cudaMalloc slab per context, mapped
 *           into the peers once per call with CUDA IPC handles (exchanged with one small NCCL
 *           all-gather, which is also the barrier between the factor initialisation and the
 *           first remote store).  Ordering: a kernel's peer stores are complete when it
 *           completes; the statistics exchange (a collective every rank contributes to)
 *           that follows every solve cannot finish on any rank before every rank's solve
 *           has finished, so a rank reads remote rows only after they landed, and a rank's
 *           next store into a matrix happens only after every peer has passed the exchange
 *           behind its last reader of it.  Needs <= 8 ranks on
 *           one node with peer access; if any rank cannot map a peer, every rank falls back
 *           to COLLECTIVE for the call (splatt_stats.exchange tells which ran).  Results are
 *           bit-identical to COLLECTIVE.
 * Errors: BADINPUT (unknown mode).                                                       */
enum { SPLATT_XCHG_COLLECTIVE = 0, SPLATT_XCHG_PEER = 1 };
splatt_status splatt_ctx_set_exchange(splatt_ctx* ctx, int32_t mode);

/* In-process loopback group (testing/emulation of the sharded path on ONE device): nranks
 * logical ranks, each a host thread with its own context and its own stream (a context
 * on the legacy default stream is rejected), run the same multi-rank ALS as above; the
 * exchanges go through device memory with host barriers between them (no kernel waits on
 * another rank).  nranks in [1, 8].  Destroy the group after every rank has finished.    */
splatt_status splatt_loopback_create(int32_t nranks, splatt_loopback** out);
splatt_status splatt_ctx_set_comm_loopback(splatt_ctx* ctx, splatt_loopback* group,
                                           int32_t rank);
void          splatt_loopback_destroy(splatt_loopback* group);

/* Host-only (no device needed): cut S slices with nnz weights w[0..S) into G
 * contiguous ranges minimising the maximum range weight;
 * boundaries leftmost-greedy under the optimal cap.  bounds: G+1 entries,
 * bounds[0] = 0, bounds[G] = S.  G >= 1.                                          */
splatt_status splatt_partition(const uint64_t* w, uint64_t S, int32_t G, uint64_t* bounds);

/* Host-only: the SPLATT_PART_NNZ split of slices with nnz weights w[0..S) among G ranks.
 * row_bounds (G+1): rank g owns rows [row_bounds[g], row_bounds[g+1]); split (G-1
 * capacity): the split slices, ascending, *nsplit of them; share: rank `rank`'s nonzeros =
 * whole slices [full_lo, full_hi) plus, for each of npart partial slices, the nonzeros whose
 * rank within that slice (input order) lies in [part_begin, part_end).  Any output may be
 * NULL.  Errors: BADINPUT (G < 1, rank out of range, S > 0 with w NULL).               */
typedef struct {
  uint64_t full_lo, full_hi;
  int32_t  npart;
  uint64_t part_slice[2], part_begin[2], part_end[2];
} splatt_nnz_share;
splatt_status splatt_partition_nnz(const uint64_t* w, uint64_t S, int32_t G, int32_t rank,
                                   uint64_t* row_bounds, uint64_t* split, uint64_t* nsplit,
                                   splatt_nnz_share* share);

/* Bitwise-reproducible ROOT MTTKRP (SURVEY.md §8(b) "Determinism"): a root slice cut by a
 * chunk seam gets its partial rows added with fp64 atomics by default, so the rounding of
 * those rows (and of the ALS built on them) can differ run to run.  With `on` the partial rows
 * are kept per chunk and summed by two more kernels in an order fixed by the slice's chunk
 * span; every result of the ALL policy is then bitwise reproducible (the dense steps
 * already reduce in fixed order).  INTERNAL/LEAF traversals (ONE/TWO) keep their
 * reductions at L2 and are not covered.  Cost: c2 MTTKRP +13%, c4 +1.5%.
 * Errors: BADINPUT (NULL).                                                              */
splatt_status splatt_ctx_set_deterministic(splatt_ctx* ctx, int32_t on);

/* Leaf-mode tiling of the ROOT MTTKRP (the mode tiling the paper's
 * port omits).  When the leaf factor of a tree (I_leaf x ld doubles)
 * exceeds l2_fraction x the L2 capacity, the tree is split once (on first use, at the rank
 * the MTTKRP runs with) into T = ceil(bytes / (l2_fraction x L2)) trees by leaf-id range,
 * run one after another (later tiles add into the owned rows), so each tile's leaf rows
 * stay in L2.  It trades DRAM misses for split fibers (more internal-node gathers) and a
 * one-time split (c3: ~5 ms per tree, 100M nonzeros): on c3 (480k-row leaf factor,
 * 138 MB) the 20-iteration ALS MTTKRP drops 269 -> 247 ms.
 * l2_fraction = SPLATT_LEAF_TILING_AUTO (the default): tiles of half the L2 inside
 * splatt_cpd_als* runs of >= 10 iterations (where the split pays for itself), none for a
 * single splatt_mttkrp; 0 = off; > 0 = always, at that fraction.
 * Errors: BADINPUT (> 4, or negative other than AUTO).                                  */
#define SPLATT_LEAF_TILING_AUTO (-1.0)
splatt_status splatt_ctx_set_leaf_tiling(splatt_ctx* ctx, double l2_fraction);

/* ---------------------------------------------------------------- CSF */
/* Build the CSF set of `coo` on the device (sort = PAPER.md:415).
 * The policy (SPLATT_CSF_ALL / ONE / TWO above) decides which trees are built: CSF k
 * is rooted at its root mode (ALL: CSF_n at mode n); below the root the other modes
 * follow by ascending length, ties to the lower mode id.  Level l < N-1
 * holds ids_l (the level's coordinate) and ptr_l (offsets into level l+1, one
 * extra end entry); the leaf level holds ids_{N-1} and vals in sorted order.
 * Bit-exact: the result is a pure integer function of the input.
 * nmodes and dims must equal coo->nmodes / coo->dims (they follow the north star's
 * call shape).  Errors: BADINPUT (nmodes, nnz = 0, dims, index >= dim, unknown
 * policy, mismatch), UNSUPPORTED (nnz >= 2^31: 32-bit leaf positions and sort counts). */
splatt_status splatt_csf_build(splatt_ctx* ctx, const splatt_coo* coo, int32_t nmodes,
                               const uint64_t* dims, int32_t policy, splatt_csf** out);
/* Allocation of a built CSF set: *ncsf (ALL: N, ONE: 1, TWO: 2) and, for mode `mode`,
 * the CSF index `which` and the tree level `level` its MTTKRP uses (0 = ROOT, N-1 =
 * LEAF, else INTERNAL).  Any output may be NULL; `mode` must be in [0, N) unless both
 * `which` and `level` are NULL.  Host-only, synchronous.                            */
splatt_status splatt_csf_dispatch(const splatt_csf* csf, int32_t mode, int32_t* ncsf,
                                  int32_t* which, int32_t* level);
/* Shape of CSF `which` (0..ncsf-1): mode_perm[0..N) (level -> mode) and n_nodes[l]
 * per level; either may be NULL.  Synchronous, host outputs.                       */
splatt_status splatt_csf_info(const splatt_csf* csf, int32_t which, int32_t* nmodes,
                              int32_t* mode_perm, uint64_t* n_nodes);
/* Copy level `level` of CSF `which` to HOST buffers (any may be NULL): ids
 * (n_nodes[level]), ptr (n_nodes[level]+1; levels < N-1 only), vals (nnz; leaf
 * level only).  Synchronous.  For bit-exact tests.                                 */
splatt_status splatt_csf_export(const splatt_csf* csf, int32_t which, int32_t level,
                                uint32_t* ids, uint32_t* ptr, double* vals);
void          splatt_csf_free(splatt_csf* csf);

/* ---------------------------------------------------------------- MTTKRP */
/* out[i, r] = sum over nonzeros p with ind_mode[p] = i of
 *             v_p * prod_{m != mode} factors[m][ind_m[p] * ld + r]      (C-6)
 * for every i < dims[mode], r < rank; rows with no nonzeros are written 0; columns
 * r >= rank of `out` are written 0.  factors: N device pointers (factors[mode] is
 * ignored, may be NULL), each dims[m] x ld.  out: device, dims[mode] x ld.
 * Uses the CSF and kernel the build policy assigns to `mode` (splatt_csf_dispatch).
 * ROOT results are deterministic; INTERNAL/LEAF (policies ONE/TWO) accumulate with
 * fp64 atomics, so their rounding order varies run to run.  A CSF set keeps per-tree
 * MTTKRP scratch (chunk tables, seam rows, hot-row lists, leaf tiles) built on first use:
 * use a set from one context / stream at a time.  Errors: BADINPUT (mode,
 * rank not in [1,128],
 * ld < rank, NULL pointers).  Asynchronous on the context stream.                  */
splatt_status splatt_mttkrp(splatt_ctx* ctx, const splatt_csf* csf, int32_t mode,
                            const double* const* factors, int32_t rank, int32_t ld,
                            double* out);

/* As splatt_mttkrp, on CSF `which` of the set (0..ncsf-1) instead of the policy's
 * choice: the kernel kind follows the level of `mode` in that CSF (ROOT / INTERNAL /
 * LEAF) — the configuration override of SPEC.md:168, used to test every kernel on every
 * tree.  Errors: as splatt_mttkrp, plus BADINPUT for `which` out of range.            */
splatt_status splatt_mttkrp_csf(splatt_ctx* ctx, const splatt_csf* csf, int32_t which,
                                int32_t mode, const double* const* factors, int32_t rank,
                                int32_t ld, double* out);

/* ---------------------------------------------------------------- CP-ALS */
/* Algorithm 1 for an N-mode tensor, fixed readings DESIGN.md §2:
 * factors initialised U[0,1) by counter-based splitmix64 from `seed` (C-2); per
 * iteration, per mode n: V = *_{m!=n} G_m, M = MTTKRP_n, A_n = M V^-1 by Cholesky
 * (ridge retry, C-7), column norms into lambda (2-norm in iteration 1, max(1,|.|max)
 * later, C-8), Gram refresh; then the fit (C-10); stop when it >= 2 and
 * |fit - fit_prev| < tol, or at max_iters (tol = 0: exactly max_iters).  Returned
 * factors have unit 2-norm columns with the norms folded into lambda (C-12).
 * Errors: BADINPUT (as csf_build; rank not in [1,128]; max_iters < 1; tol < 0 or
 * NaN), EMPTY (||X|| = 0), SINGULAR.  Synchronous.                                  */
splatt_status splatt_cpd_als(splatt_ctx* ctx, const splatt_coo* coo, int32_t rank,
                             int32_t max_iters, double tol, uint64_t seed,
                             splatt_kruskal* out);
/* As splatt_cpd_als, plus: init_factors (NULL = seeded init; else N pointers,
 * host or device, I_n x rank, ld = rank, used as the initial A_n), policy
 * (SPLATT_CSF_ALL / ONE / TWO: which CSFs are built and which MTTKRP kernel each mode
 * runs; the result differs only by rounding), stats (NULL or filled; see splatt_stats).
 * A sharded context (splatt_ctx_set_comm*) requires SPLATT_CSF_ALL (UNSUPPORTED
 * otherwise: row ownership per rank needs a ROOT traversal for every mode).          */
splatt_status splatt_cpd_als_ex(splatt_ctx* ctx, const splatt_coo* coo, int32_t rank,
                                int32_t max_iters, double tol, uint64_t seed,
                                const double* const* init_factors, int32_t policy,
                                splatt_kruskal* out, splatt_stats* stats);

/* ------------------------------------------------------- .tns ingestion and statistics
 * the paper's datasets are FROSTT .tns files.
 * Format: one nonzero per line, N 1-based integer indices then a decimal
 * value, whitespace separated; '#' comment lines and blank lines are skipped; N is the field
 * count of the first data line minus one (1..8); dims[m] = the largest index seen in mode
 * m; duplicates are kept in file order.  Host-only (no device needed).                    */
typedef struct splatt_tensor splatt_tensor;  /* host COO owned by the library           */

/* Parse `path` (multi-threaded, file order preserved) into *out.  Errors: BADINPUT
 * (unreadable file, no nonzeros, wrong field count, non-integer index, index < 1 or >= 2^32,
 * non-numeric value: the message, splatt_tensor_error(), names the 1-based line), NOMEM.   */
splatt_status splatt_tns_read(const char* path, splatt_tensor** out);
/* A splatt_coo view of t (host pointers into t; valid until splatt_tensor_free).           */
splatt_status splatt_tensor_coo(const splatt_tensor* t, splatt_coo* view);
void          splatt_tensor_free(splatt_tensor* t);
/* Message of the last failed splatt_tns_read / splatt_tns_write on this thread.           */
const char*   splatt_tensor_error(void);
/* Write a HOST COO as .tns (1-based; values in shortest round-trip decimal).  nmodes 1..8.  */
splatt_status splatt_tns_write(const char* path, const splatt_coo* coo);

/* Table I statistics of a HOST COO: dims, nnz, density =
 * nnz / prod(dims) in floating point, and per mode the non-empty slices and the largest
 * slice (nonzeros sharing one index).  Errors: BADINPUT (index >= dim, NULL).              */
typedef struct {
  int32_t  nmodes;
  uint64_t nnz;
  uint64_t dims[SPLATT_MAX_NMODES];
  double   density;
  uint64_t nonempty_slices[SPLATT_MAX_NMODES];
  uint64_t max_slice_nnz[SPLATT_MAX_NMODES];
} splatt_tensor_stats;
splatt_status splatt_coo_stats(const splatt_coo* coo, splatt_tensor_stats* out);

/* ------------------------------------------------------- CP-ALS on a prebuilt CSF set
 * As splatt_cpd_als_ex, on the trees of a splatt_csf_build result (its policy decides the
 * kernels): the build ("Sort") and the COO validation are skipped, so repeated runs on one
 * tensor (rank sweeps, restarts with other seeds) pay for them once.  ||X||^2 is summed over
 * the tree's leaf values (another order than the COO's: rounding-level difference).  Not
 * with a sharded context (UNSUPPORTED).  Errors: as splatt_cpd_als_ex.                  */
splatt_status splatt_cpd_als_csf(splatt_ctx* ctx, const splatt_csf* csf, int32_t rank,
                                 int32_t max_iters, double tol, uint64_t seed,
                                 const double* const* init_factors, splatt_kruskal* out,
                                 splatt_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* SPLATT_B200_H */
