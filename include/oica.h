/*
 * oica.h -- C ABI of liboica.so, the B200 (sm_100a) hot path of Fast Ordering ICA
 * (Matsuda & Yamaguchi, "Efficient Estimation of Unique Components in ICA by Matrix
 * Representation", arXiv 2408.17118).  Citations "PAPER.md:n" are lines of the paper's
 * LaTeX source; readings Ann are listed in DESIGN.md §2.
 *
 * The library computes, for each component i = 1..N_out (Alg. 2):
 *   draw L candidate rows, project them orthogonal to the accepted
 *   rows (E = W^T W, w <- w - E w) and normalise; then iterate
 *     Z = B X,  B <- (Z o Z o Z) X^T / M - 3 B,
 *     project, normalise, drop converged rows
 *   and accept the candidate of largest Upsilon(alpha), alpha = sum z^4 / M - 3
 *   (eqs. (1)-(2), :257-259, :264).
 *
 * Conventions (all functions):
 *   - Every function returns oica_status; no C++ exception crosses the ABI.
 *     oica_last_error(ctx) holds a message until the next call on ctx.
 *   - "device" pointers are CUDA global-memory addresses on the context's device;
 *     "host" pointers are ordinary CPU memory.  Matrices are ROW-MAJOR.
 *   - The caller owns every buffer it passes and allocates every output; the library
 *     never frees caller memory and retains no host pointer after a call returns.
 *     Device inputs passed to oica_set_data are BORROWED until the next set_data /
 *     destroy; all derived operands and workspace are owned by the context.
 *   - CUDA / NCCL failures return OICA_ERR_CUDA / OICA_ERR_NCCL and leave the context
 *     usable only for oica_destroy.
 *   - A context is single-threaded: one context per device and rank.
 *   - The library works on the context's stream (cfg->stream, or its own non-blocking stream)
 *     and does not order itself after other streams: device inputs must be complete when a
 *     call is made (the Python binding synchronizes torch's current stream before passing one).
 *   - With world > 1 every call that computes is COLLECTIVE: all ranks call it with
 *     identical scalar arguments.
 */
#ifndef OICA_H_
#define OICA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oica_ctx oica_ctx;

typedef enum {
  OICA_OK = 0,
  OICA_ERR_INVALID_ARGUMENT = 1,      /* bad size, NULL pointer, out-of-range parameter      */
  OICA_ERR_DIMENSION_MISMATCH = 2,    /* shapes inconsistent with the data set on the ctx     */
  OICA_ERR_RANK_DEFICIENT = 3,        /* whitening: covariance eigenvalue < floor (A11)       */
  OICA_ERR_ALL_CANDIDATES_DEGENERATE = 4, /* every candidate projected to ||w|| < 1e-12 (A18)  */
  OICA_ERR_DOMAIN = 5,                /* no eligible candidate has alpha > -2 (eq. (1), A13)  */
  OICA_ERR_STATE = 6,                 /* call order violated (e.g. extract before set_data)   */
  OICA_ERR_UNSUPPORTED_DEVICE = 7,    /* device is not compute capability 10.0 (sm_100a)      */
  OICA_ERR_OUT_OF_MEMORY = 8,
  OICA_ERR_CUDA = 9,
  OICA_ERR_NCCL = 10,
  OICA_ERR_NONFINITE = 11             /* a candidate update was not finite (non-finite data);  */
                                      /* the extraction stops instead of dropping the row      */
} oica_status;

/* Arithmetic of the fixed-point contraction (the two products of PAPER.md:243-245). */
typedef enum {
  OICA_PREC_AUTO = 0,   /* TC when M_global >= 16384, else FP32               */
  OICA_PREC_FP32 = 1,   /* FP32 FFMA on CUDA cores, fp32 accumulate per flush, fp64 slots    */
  OICA_PREC_TC = 2,     /* tcgen05 tensor cores: fp16 X, one-pass fp16 GEMM1 on w_h =        */
                        /* fp16(2^4 w)/2^4 with eq. (5)'s -3w evaluated at w_h (consistent),  */
                        /* rows whose step stagnates near the fp16 floor promoted to the      */
                        /* two-pass w_h + w_l operand; fp16 GEMM2; fp32 TMEM accumulation,    */
                        /* fp64 across slots                                   */
  OICA_PREC_TC_SPLIT = 3 /* as TC with every row two-pass from the start (w to ~2^-22)        */
} oica_precision;

/* Multi-GPU partitioning.  world == 1 ignores it. */
typedef enum {
  OICA_SHARD_L = 0,     /* candidates split over ranks, X replicated, one exchange/component; */
                        /* ranks iterate in lock step (4-byte count all-reduce per iteration) */
  OICA_SHARD_M = 1,     /* samples split over ranks, fp64 allreduce of G, s4 per iteration   */
  OICA_SHARD_HYBRID = 2 /* L-shard until the global active count falls to OICA_HYBRID_ROWS     */
                        /* (env; default 128 x world): the remaining runs are all-gathered,    */
                        /* iterated M-sharded over the replicated X (fp64 allreduce per         */
                        /* iteration) and handed back to their owners.   */
                        /* Equal to L-shard within tolerance (the tail sums ranks in NCCL       */
                        /* order), not bitwise.                                                 */
} oica_shard_mode;

typedef struct {
  int32_t device;            /* CUDA device ordinal                                         */
  int32_t rank;              /* 0 <= rank < world                                           */
  int32_t world;             /* number of ranks (1 = single GPU)                            */
  int32_t shard_mode;        /* oica_shard_mode                                             */
  int32_t precision;         /* oica_precision                                              */
  int32_t reserved;
  void* stream;              /* cudaStream_t to run on, or NULL: the context creates one    */
  const void* nccl_unique_id;/* 128-byte ncclUniqueId from oica_nccl_unique_id (world > 1)  */
} oica_config;

/* Per-component results, caller-allocated HOST arrays of length >= N_out (W: N_out x N). */
typedef struct {
  double* W;              /* accepted rows, canonical sign (A17), whitened coordinates       */
  double* alpha;          /* alpha_q = sum_m y^4/M - 3 at the accepted w (eq. (2), A15)      */
  double* upsilon;        /* Upsilon(alpha_q) (eq. (1))                                      */
  int64_t* index;         /* q: global candidate id accepted (cluster minimum, A6)            */
  int32_t* iters;         /* fixed-point updates applied to candidate q                      */
  int32_t* n_iter;        /* iterations executed for the component (max over candidates)     */
  int32_t* cluster_size;  /* eligible candidates on q's fixed point (1-|cos| <= 1e-6)        */
  int32_t* n_converged;   /* candidates that met the convergence test (A1/A2)                */
  int32_t* n_unconverged; /* candidates still active at the cap K (A4)                       */
  int32_t* n_degenerate;  /* candidates with ||w|| < 1e-12 after a projection (A18)          */
  int64_t* sum_active;    /* sum over iterations of active rows (algorithmic-work counter)   */
  uint8_t* gaussian_flag; /* Upsilon_q < 2(N-i+2)(N-i+1)/M                    */
  uint8_t* near_tie;      /* best and second-best clusters within 1e-6 relative (A6)         */
  int32_t n_extracted;    /* rows written (< N_out only with OICA_STOP_ON_GAUSSIANITY)       */
  int32_t stopped;        /* 1 if the Gaussianity test ended extraction   */
  int32_t* dim;           /* dimension the component's iteration ran in: N, or N-i+1 with   */
                          /* OICA_REDUCE_X (algorithmic work = sum_active (4 dim M + 3 M))   */
  double* objective;      /* sum_m y^4 / M at the accepted w (the quantity alpha + 3 of eq. (2), */
                          /* the north_star's objective), from the exact fp64 pass            */
} oica_result;

/* Flags for oica_extract_components. */
#define OICA_INCLUDE_UNCONVERGED 0x1u  /* rows still active at K join the argmax (A4, Alg. 1)   */
#define OICA_STOP_ON_GAUSSIANITY 0x2u  /* break on the Gaussianity test     */
#define OICA_RAW_ARGMAX          0x4u  /* accept p = argmax itself, no cluster rule (A6)        */
/* §3.3 reduction (Alg. 2 lines 4-12 and 28): component
 * i iterates on X~ = G X (d = N-i+1 rows, G an orthonormal basis of the complement of the
 * accepted rows) instead of projecting every update; candidates start at b0 = G r/||G r|| (A9),
 * the accepted row is w = G^T b.  Same trajectories as the default projection form in exact
 * arithmetic; 4 d M instead of 4 N M flop per row-iteration. */
#define OICA_REDUCE_X            0x8u
/* Host-launched iterations.  By default, on one rank, where an iteration is short next to a host
 * round trip (M x padded N < 1e8: the device-side loop of DESIGN.md §5 "iteration"), the
 * do-while of PAPER.md:241-256 runs on the device as one CUDA-graph WHILE loop per component
 * (bitwise the same results); OICA_EAGER launches every iteration from the host instead, which
 * times each step launch for oica_get_iteration_log / oica_stats.step_ms. */
#define OICA_EAGER               0x10u
/* Tiny FP32 problems (L <= 512, M < 65536, one rank) run the device-side loop as ONE cooperative
 * kernel whose grid barriers need its blocks co-resident; several extractions running concurrently
 * on one GPU (one context / stream each) are better served by the CUDA-graph loop: this flag
 * selects it (bitwise the same results). */
#define OICA_NO_PERSISTENT       0x20u

/* Counters of the last extract / step call (for benchmarks; all host values). */
typedef struct {
  int64_t kernel_launches;   /* kernels launched by the library since the last reset        */
  int64_t step_launches;     /* launches of the fused fixed-point kernel                    */
  double step_ms;            /* summed CUDA-event time of those launches                    */
  double step_flops;         /* algorithmic flops of those launches: sum L_act (4NM + 3M)   */
  int64_t iterations;        /* fixed-point iterations executed                             */
  int64_t sum_active;        /* sum over iterations of active rows                           */
  int32_t precision;         /* precision actually used by the step kernel                  */
  int32_t slots;             /* split-M slots S                                             */
  double step_issued_flops;  /* flops the step launches issued to the tensor pipe / FMA units,*/
                             /* padding and second passes included (row tiles x NP)         */
  int64_t fine_rows;         /* sum over step launches of rows run with the two-pass GEMM1   */
  int64_t tail_iterations;   /* iterations run in the hybrid tail (OICA_SHARD_HYBRID)        */
  double exchange_ms;        /* CUDA-event time of the NCCL exchanges on the context stream  */
  int64_t exchange_calls;    /* NCCL collectives issued (0 without a communicator)          */
  int64_t graph_iterations;  /* iterations run by the device-side loop (not in step_ms/step_flops) */
  double graph_ms;           /* CUDA-event time of those loops (steps and updates together)  */
  double graph_flops;        /* algorithmic flops of those iterations: sum L_act (4NM + 3M)  */
} oica_stats;

/* ---- lifetime ---------------------------------------------------------------------- */

/* Create a context on cfg->device.  Fails with OICA_ERR_UNSUPPORTED_DEVICE unless the device
 * is compute capability 10.0.  world > 1 initialises an NCCL communicator from
 * cfg->nccl_unique_id (collective over all ranks).  With a communicator every host wait of the
 * library polls NCCL's asynchronous error state and gives up after OICA_NCCL_TIMEOUT_S seconds
 * (environment, default 900): the communicator is aborted, the call returns OICA_ERR_NCCL and
 * the context is usable only for oica_destroy (a dead or absent peer never hangs the caller). */
oica_status oica_create(const oica_config* cfg, oica_ctx** out);
oica_status oica_destroy(oica_ctx* ctx);
const char* oica_status_string(oica_status s);
const char* oica_last_error(const oica_ctx* ctx);
/* Write a fresh 128-byte ncclUniqueId into out (host); call on rank 0 and broadcast. */
oica_status oica_nccl_unique_id(void* out);

/* ---- boundary: whitening "in advance" (readings A11/A12) ---------- */

/* X_dev: device fp32 N x M raw signals, row stride ld >= M.  Computes the row means, the
 * covariance C = Xc Xc^T / M in fp64, its eigendecomposition (host Jacobi), V = D^{-1/2} E^T
 * (eigenvalues descending, each eigenvector's largest-|entry| positive) and writes
 * Xw = V (X - mean) as fp32 to Xw_dev (N x M, stride ld_out >= M).  mean_out (N), V_out (N x N),
 * eig_out (N) are host fp64 and may be NULL.  RANK_DEFICIENT if min eig < eig_floor * max eig. */
oica_status oica_whiten(oica_ctx* ctx, const float* X_dev, int64_t N, int64_t M, int64_t ld,
                        double eig_floor, float* Xw_dev, int64_t ld_out,
                        double* mean_out, double* V_out, double* eig_out);

/* ---- data and candidates --------------------------------------------------------------- */

/* Bind whitened data: Xw_dev device fp32 N x M_local (stride ld >= M_local), BORROWED.
 * M_global is the total sample count M of eq. (2) (== M_local unless shard_mode = M).
 * 1 <= N <= 256, M_global > N.  Prepares the context-owned operand planes. */
oica_status oica_set_data(oica_ctx* ctx, const float* Xw_dev, int64_t N, int64_t M_local,
                          int64_t ld, int64_t M_global);
/* Same with a HOST fp32 source: the library copies it into an owned device buffer (the
 * end-to-end entry point).  The copy is ENQUEUED, not finished, when the call returns: it runs
 * on a second stream in pieces of whole slots and the first step of the next extraction starts
 * on each piece as it lands.  A pageable source may be reused as soon as the
 * call returns (the CUDA runtime stages it); a PINNED (page-locked) source must stay valid and
 * unchanged until the next oica_extract_components / oica_synchronize / oica_set_data* call on
 * this context returns. */
oica_status oica_set_data_host(oica_ctx* ctx, const float* Xw_host, int64_t N, int64_t M_local,
                               int64_t ld, int64_t M_global);

/* C3: distribute whitened data from rank `root` to every rank (collective; every
 * rank passes the same N, M_global, root).  X_root: root's device fp32 N x M_global (stride
 * ld_root), ignored on the other ranks (may be NULL there).  X_out: this rank's device buffer,
 * N x M_local with stride ld_out >= M_local, where M_local = M_global for OICA_SHARD_L / HYBRID
 * (X replicated: one ncclBroadcast, or one per row when a stride is not M_global; on root X_out
 * may equal X_root) and the samples [rank M/world, (rank+1) M/world) for OICA_SHARD_M (root sends
 * every rank its columns, row by row, with ncclSend/ncclRecv).  Without a communicator it is a
 * device copy.  Synchronous.  The result is what oica_set_data then borrows. */
oica_status oica_distribute_data(oica_ctx* ctx, const float* X_root, int64_t N, int64_t M_global, int64_t ld_root,
                                 float* X_out, int64_t ld_out, int32_t root);

/* Fix the candidate generator (seed) and the global candidate count L (PAPER.md:126, :136,
 * :237; readings A7/A8).  Candidates are drawn afresh for every component from the
 * counter-based generator of DESIGN.md §2 A7, keyed by (seed, i, global id l, coordinate).
 * L-shard: rank r owns ids [r*L/world, (r+1)*L/world).  1 <= L < 2^24. */
oica_status oica_init_candidates(oica_ctx* ctx, uint64_t seed, int64_t L);

/* ---- the hot path ---------------------------------------------------------------------- */

/* Extract components k_prefix+1 .. N_out (Alg. 2 with the projection of Alg. 1).
 * max_iter = K >= 1 (do-while, A19); tol > 0 is the convergence test 1 - |w . w_prev| <= tol
 * (A1/A2; the paper's chord eps corresponds to tol = eps^2/2).  W_prefix (host fp64
 * k_prefix x N, orthonormal rows, may be NULL when k_prefix == 0) seeds the accepted rows
 * (resume / teacher forcing).  Writes rows k_prefix .. n_extracted-1 of out (synchronous).
 * With world > 1 the call is collective: every rank passes the same arguments (checked by a
 * hash all-reduce; a mismatch returns INVALID_ARGUMENT on every rank).
 * Errors: ALL_CANDIDATES_DEGENERATE, DOMAIN, INVALID_ARGUMENT (N_out outside [k_prefix+1, N]). */
oica_status oica_extract_components(oica_ctx* ctx, int32_t N_out, int32_t max_iter, double tol,
                                    uint32_t flags, const double* W_prefix, int32_t k_prefix,
                                    oica_result* out);

/* ---- test and benchmark entry points ---------------------------------------------------- */

/* One fused contraction (PAPER.md:243-244 before the -3B term) on caller rows:
 * W_dev device fp64 L x N (unit rows); outputs device fp64 G_dev (L x N) = sum_m y^3 x^T and
 * s4_dev (L) = sum_m y^4 with y = w X, summed over the local samples in the context's precision
 * and slot order.  (Uses the context's workspace; L <= the L of init_candidates.) */
oica_status oica_fixed_point_step(oica_ctx* ctx, const double* W_dev, int64_t L,
                                  double* G_dev, double* s4_dev);
/* The same contraction with a per-row precision (tensor-core contexts): fine_host
 * (host, L bytes) marks the rows evaluated in two-pass "fine" precision; they must follow every
 * coarse row (the order the runtime's compaction keeps), else INVALID_ARGUMENT.  A row's result
 * does not depend on the rows it shares a 128-row tile with.  FP32 contexts ignore fine_host. */
oica_status oica_fixed_point_step_mixed(oica_ctx* ctx, const double* W_dev, int64_t L, const uint8_t* fine_host,
                                        double* G_dev, double* s4_dev);
/* The candidate generator + projection + normalisation
 * for component i (1-based) against host W_acc (k x N, may be NULL if k == 0):
 * writes this rank's L_local x N fp64 rows to W_dev (device).  Degenerate rows are zero. */
oica_status oica_draw_candidates(oica_ctx* ctx, int32_t i, const double* W_acc, int32_t k,
                                 double* W_dev);
/* End state of the last extracted component's candidates on this rank (host outputs, each
 * L_local long, any may be NULL): W (L_local x N fp64), alpha at the last forward pass,
 * iterations, state (0 active/unconverged, 1 converged, 2 degenerate). */
oica_status oica_get_candidates(oica_ctx* ctx, double* W, double* alpha, int32_t* iters,
                                uint8_t* state, int64_t* L_local, int64_t* id_base);
/* Per-iteration log of the last oica_extract_components call: one record per
 * executed fixed-point iteration of every component on this rank.  step_ms is the CUDA-event
 * time of that iteration's step launch(es) on the context stream (-1 for iterations of the
 * device-side loop, which are not timed one by one: use OICA_EAGER); flops its algorithmic work
 * L_act (4 d + 3) M_local (d = the dimension iterated on).  Copies min(cap, *n) records;
 * *n = the number available (call with cap = 0 to size). */
typedef struct {
  int32_t component;   /* 1-based i                                                           */
  int32_t iteration;   /* t (1-based)                                                         */
  int32_t L_act;       /* active runs entering the iteration                                  */
  int32_t fine_rows;   /* of which run in two-pass precision                                  */
  double step_ms;
  double flops;
} oica_iteration_record;
oica_status oica_get_iteration_log(oica_ctx* ctx, oica_iteration_record* out, int64_t cap, int64_t* n);
oica_status oica_get_stats(oica_ctx* ctx, oica_stats* out);
oica_status oica_reset_stats(oica_ctx* ctx);
/* Synchronise the context's stream (for host-side timing). */
oica_status oica_synchronize(oica_ctx* ctx);

/* ---- host-only selection merge (multi-GPU decision; also unit-tested on CPU) ------------ */

/* One candidate cluster as reported by a rank: its minimum global id q, the accepted
 * quantities of that member and the cluster's local size.  w is N doubles. */
typedef struct {
  double upsilon;
  double alpha;
  int64_t q;
  int64_t size;
  int32_t iters;
  int32_t valid;          /* 0 = empty slot */
  double objective;       /* sum y^4 / M of member q (alpha + 3)                             */
} oica_cluster_record;
/* Host-only helpers of OICA_REDUCE_X (pure functions, no device).  oica_complement_basis: W is
 * k x N with orthonormal rows (k < N); writes G, (N-k) x N, rows orthonormal and orthogonal to
 * every row of W (the last N-k columns of Q in the Householder QR of W^T).  oica_deflate_basis:
 * G is d x N with orthonormal rows, b a unit d-vector; writes the (d-1) x N basis of the
 * complement of w = G^T b inside span(G) (rows 2..d of H G, H the reflection taking b to -+e1). */
oica_status oica_complement_basis(const double* W, int32_t k, int32_t N, double* G);
/* Host-only: the split-M slot plan of the step kernels (DESIGN.md §5 "HBM layout").  Slot length
 * depends on M_global and the precision only (so every row's fp32-per-slot / fp64-across-slot
 * arithmetic is the same for any GPU count, tiling or active-set size): a multiple of 384 samples
 * for the tensor-core step; for the FP32 step below 65536 samples, up to 128 slots of >= 128
 * samples, 64-aligned.  precision: an oica_precision (AUTO resolves as oica_set_data does).
 * S_local = ceil(M_local / slot_len) slots cover this rank's samples. */
oica_status oica_slot_plan(int32_t precision, int64_t M_global, int64_t M_local, int64_t* slot_len,
                           int32_t* S_local);
/* Host-only: split-slot parts of the tensor-core step (DESIGN.md §5 "few active rows") when
 * L_global runs are active over S slots: P in [1, 8] CTAs share each slot's chunks.  A function
 * of (L_global, S) only; P > 1 only while round_up(ceil(L_global/128), 2) * S <= 148. */
oica_status oica_split_parts(int32_t L_global, int32_t S, int32_t* P);
oica_status oica_deflate_basis(double* G, int32_t d, int32_t N, const double* b, double* G_out);

/* Merge n records (from all ranks, records[k].w = w + k*N) into the global decision of
 * reading A6: records whose rows satisfy 1 - |w_a . w_b| <= 1e-6 are one cluster (sizes add,
 * q = minimum id, its record supplies alpha/upsilon/iters/w); the winner is the cluster of
 * largest upsilon (ties -> lowest q); near_tie if the runner-up is within 1e-6 relative.
 * Host pointers; pure function (the device accept kernel runs the same source).  Writes the
 * winner's index into `records` to *winner and the merged size / near-tie flag. */
oica_status oica_merge_records(const oica_cluster_record* records, const double* w, int32_t n,
                               int32_t N, int32_t* winner, int64_t* merged_size,
                               uint8_t* near_tie);

#ifdef __cplusplus
}
#endif
#endif /* OICA_H_ */
