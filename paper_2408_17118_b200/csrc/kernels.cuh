// Launch wrappers of the liboica kernels (internal).  Every wrapper enqueues on `st` and
// returns the number of kernels it launched (for the launch counter in oica_stats).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace oica {

// ---- K1: candidate draw + projection + normalisation
// Also resets the per-candidate precision state: fine[j] = fine_init, dprev[j] = +inf.
int launch_cand_init(cudaStream_t st, uint64_t seed, int i, int64_t id_base, int64_t L_local, int N,
                     const double* Wacc, int k, double* W64, uint8_t* state, uint8_t* keep, uint8_t* fine,
                     uint8_t fine_init, double* dprev);

// ---- K4: order-preserving compaction of the active set
// act_in == nullptr means the identity list.  Kept rows are stably partitioned: coarse rows
// first, then rows with fine[id] != 0 (fine may be null).  Writes act_out, out_dev[0] = L_act,
// out_dev[1] = number of coarse rows, and the same two ints to host_mapped (may be null).
// cnt_in (device, may be null): the true L_in (L_in is then an upper bound); hist (may be null):
// the new [L_act, n_coarse] pair is also appended there.
int launch_compact(cudaStream_t st, const int* act_in, const uint8_t* keep, const uint8_t* fine, int L_in,
                   int* act_out, int* out_dev, int* host_mapped, const int* cnt_in = nullptr, int* hist = nullptr);

// Operand rows of the step kernels, stored BY CANDIDATE ID (row l at l * NP): the step kernels
// gather the rows of their active positions through the active list, and the fused update
// (launch_update) rewrites a row whenever it updates that candidate.  These two build rows
// 0..L-1 from the fp64 master (after the candidate draw; for oica_fixed_point_step).
int launch_operand_f32(cudaStream_t st, int L, const double* W64, int N, int NP, float* W32);
// Split-fp16 operand (TC path): hi = fp16(2^4 w), lo = fp16(2^4 w - hi) for fine rows, 0 for
// coarse rows (fine == null: all rows fine).
int launch_operand_f16x2(cudaStream_t st, int L, const double* W64, int N, int NP, const uint8_t* fine, __half* Whi,
                         __half* Wlo);

// ---- K2b: fused GEMM-cube-GEMM on CUDA cores (PAPER.md:243-245 before the -3B term)
// Gp[s][a][n] (stride ldg = NP), s4p[s][a] over slots s of slot_len samples.
// act (device): the active list; position a uses operand row act[a] (W32 by candidate id).
int launch_step_simt(cudaStream_t st, const float* X, int64_t ld, int64_t M, int N, int NP,
                     const float* W32, const int* act, int L_act, int64_t slot_len, int S, int flush,
                     double* Gp, double* s4p, int64_t cap, const int* cnt);

// Slot partials of the step kernel: fp64 (SIMT) or fp32 (tensor cores: the exact TMEM value).
struct SlotPartials {
  const void* p;
  bool f32;
  // split-slot parts (f32 only, common.cuh split_parts): when P = split_parts(L_g, S) > 1 the
  // partial of (slot s, part q, row a) is sub[((s kSplitMax + q) sub_cap + a) ldg + n], q < P;
  // L_g = *cnt_g (device) or L_g_host (cnt_g null).  sub null: always P = 1.
  const float* sub = nullptr;
  int64_t sub_cap = 0;
  const int* cnt_g = nullptr;
  int L_g_host = 0;
};
// The point the contraction was evaluated at: the operand rows, BY CANDIDATE ID (stride ld): the
// -3w term and the alpha~ identity use it so eq. (5) is evaluated consistently.
// f16: (hi + lo) / 2^4 (lo may be null); f32: W32; all null: the fp64 master row.  The fused
// update reads a row's point and then overwrites the row with the next iteration's operand.
struct EvalPoint {
  __half* hi;
  __half* lo;
  float* f32;
  int ld;
};

// Device iteration state of a context (DESIGN.md §5 "iteration"): t = the 1-based iteration the
// next update applies (advanced by the update's last block when the iteration had active runs),
// k = accepted rows the updates project against (0 in the reduced space), done = block tickets of
// the running update (reset by its last block), sum_active = the component's algorithmic-work
// counter.  Kept on the device so an iteration needs no host argument that changes (CUDA graph)
// and a component needs no host round trip before its selection.
struct IterCtl {
  int t;
  int k;
  unsigned done;
  int pad;
  long long sum_active;   // sum over executed iterations of the active rows entering them
};

// ---- K3: fp64 epilogue: slot sum, /M - 3w, projection, normalise, convergence
// Precision promotion (TC): an unconverged row becomes fine when its step
// distance d <= d_promote stagnates (d > ratio d_prev) or t >= t_force.  fine may be null.
// nonfinite (device counter, may be null): rows whose update g was not finite (an fp16 range
// failure or non-finite data) are counted there and retired as degenerate, never silently kept
// iterating; the runtime fails the extraction with OICA_ERR_NONFINITE when the count is > 0.
struct Promotion {
  uint8_t* fine;
  double* dprev;
  double d_promote;
  double ratio;   // stagnation: d > ratio * d_prev
  int t_force;
  int* nonfinite = nullptr;
};
// K3 + K4 fused: one launch per iteration after the step (DESIGN.md §5 "iteration").  For the
// L_in = min(L_ub, cnt_in[0]) active positions: the fixed-order slot sum of G (and s4), eq. (5) at
// the evaluation point, projection against ctl->k rows of Wacc, normalisation, convergence test,
// promotion, the new master row W64[l] and the next operand row (by id); then the LAST block to
// finish compacts act_in -> act_out (kept coarse rows, then kept fine rows), writes cnt_out =
// [L_act, n_coarse] (and host_mapped, hist[2t..2t+1] if given), copies act_out back over act_in
// when copy_back (a fixed active-list buffer: CUDA-graph iterations), and advances ctl->t.
// cnt_in may alias cnt_out (every block reads it before the last block writes it).
struct UpdateArgs {
  SlotPartials G;
  const double* s4p;   // SIMT slot partials of sum y^4 (null: TC identity w_e . G)
  int S;
  int64_t cap;
  int ldg;
  EvalPoint ev;
  const int* act_in;
  int* act_out;
  int copy_back;
  int L_ub;
  const int* cnt_in;
  int* cnt_out;
  int* host_mapped;
  int* hist;
  const double* Wacc;
  int N;
  double M;
  double tol;
  double* W64;
  double* alpha_old;
  int* iters;
  uint8_t* state;
  uint8_t* keep;
  Promotion pr;
  IterCtl* ctl;
  // device-side loop (CUDA-graph WHILE nodes, one per grid-size tier): the end of the iteration
  // sets this tier's condition "more than loop_thr runs remain and t <= K_loop" and the next
  // tier's "runs remain and t <= K_loop" (loop / loop_next = 0: none)
  cudaGraphConditionalHandle loop;
  cudaGraphConditionalHandle loop_next;
  int loop_thr;
  int K_loop;
  // loop bodies unrolled U times (one WHILE re-launch per U iterations): gate_out [2] = this
  // tier's loop goes on ? (L_act, n_coarse) : (0, 0), written with the condition; gate_in (the
  // 2nd..U-th copies of the body) = the previous copy's gate_out -- 0: the loop ended inside
  // this body and the kernel returns at once (the copy's step reads the same gate as its count)
  const int* gate_in;
  int* gate_out;
  // 0: no compaction here (many rows: the caller launches k_compact, whose 1024 threads scan the
  // list faster than one block of the update could); keep[] and the row state are written
  int compact;
};
// launch_update compacts inside (last block) up to this many upper-bound rows; above, one warp per
// row updates (the HBM-bound regime) and launch_compact_iter compacts
constexpr int kUpdateCompactRows = 2048;
// ... and up to this many upper-bound rows one block per row (k_update_coop) while the row's slot
// values fit this much shared memory (S x NP x 8 bytes).  Measured: cfg 2 all components 136.7 ->
// 127.0 ms, cfg 1 22.6 -> 20.6 ms; with 2048 rows cfg 1 takes 33 ms (512-thread blocks with large
// shared memory for every mid-size iteration)
constexpr int kUpdateCoopRows = 128;
constexpr size_t kUpdateCoopSmem = 96 * 1024;
int launch_update(cudaStream_t st, const UpdateArgs& u, int NP);
// after launch_update with compact = 0: the compaction and the end of the iteration
int launch_compact_iter(cudaStream_t st, const UpdateArgs& u);
// grid-size upper bound of launch_update for L_ub rows (blocks)
int update_blocks(int L_ub, int NP);
// The whole do-while of one component for the FP32 step at tiny sizes, as ONE cooperative launch
// (k_loop_simt.cu): step units, update, compaction per iteration with grid barriers, until no run
// is active or t > K.  u: the update arguments (G = the fp64 slot partials, act_in = the active list
// kept in place, act_out = scratch, ctl, hist, ...).  NP = 32 or 64.
int launch_loop_simt(cudaStream_t st, const float* X, int64_t ld, int64_t M, int64_t slot_len, int S, int flush,
                     int K, const UpdateArgs& u, int NP, int num_sms);
// Adds the loop graph's first node: sets h = (cnt[0] > 0 && ctl->t <= K) (the first WHILE node's
// condition, so the loop also runs zero times when nothing is left to iterate)
void add_loop_gate_node(cudaGraph_t g, cudaGraphNode_t* node, cudaGraphConditionalHandle h, const int* cnt,
                        const IterCtl* ctl, int K);
// ctl <- {t, k, 0} (component start; t = 1)
int launch_ctl_set(cudaStream_t st, IterCtl* ctl, int t, int k);


// Fixed-order slot sum into G_out (L x ldo) and s4_out (L).
int launch_slot_reduce(cudaStream_t st, SlotPartials Gp, const double* s4p, int S, int64_t cap, int ldg,
                       int L, int N, double* G_out, int ldo, double* s4_out, const int* cnt = nullptr);

// alpha_old[act[a]] = s4[a] / M - 3 for a < min(L_ub, cnt[0]).
int launch_alpha_refresh(cudaStream_t st, const int* act, const int* cnt, int L_ub, const double* s4, double M,
                         double* alpha_old);

// s4 = w_eval . G (identity sum_m y^3 (w.x) = sum_m y^4), G rows by position; the evaluation point
// of position a is row act[a] (act null: a).
int launch_s4_from_g(cudaStream_t st, EvalPoint ev, const int* act, const double* G, int ldg, int L, int N,
                     double* s4, const int* cnt = nullptr);   // cnt: rows a >= cnt[0] are skipped

// ---- C4: hybrid L -> M tail: pack this rank's active rows as records
// [w (d) | alpha_old | dprev | fine | global id] (dprev, fine may be null), unpack the gathered
// records into the tail's arrays, scatter finished tail rows back to their owner by global id.
int launch_tail_pack(cudaStream_t st, const int* act, const int* cnt, int L_ub, const double* W64,
                     const double* alpha_old, const double* dprev, const uint8_t* fine, int64_t id_base, int d,
                     double* out);
int launch_tail_unpack(cudaStream_t st, const double* in, int T, int d, double* W64, double* alpha_old,
                       double* dprev, uint8_t* fine, uint8_t* state, uint8_t* keep, int64_t* ids);
int launch_tail_scatter(cudaStream_t st, int T, const int64_t* ids, const double* tW64, const double* t_alpha,
                        const int* t_iters, const uint8_t* t_state, int64_t id_base, int64_t L_local, int d,
                        double* W64, double* alpha_old, int* iters, uint8_t* state);

// ---- K5: device-side argmax, cluster assignment, exact alpha, merge + accept
struct SelectWork;  // defined in k_select.cu
struct ComponentRecord {
  double w_alpha, w_upsilon, w_objective;
  int64_t q, cluster_size, n_conv, n_unconv, n_deg, sum_active, n_nonfinite;
  int32_t iters, n_iter, status, gaussian, near_tie, n_domain;
};
struct RankSummary {
  oica_cluster_record rec[kMaxClusters];
  int64_t n_conv, n_unconv, n_deg, sum_active, n_nonfinite;
  int32_t n_iter, n_domain;
};

// Census + refinement: fills summary (per-rank records) and wsum (kMaxClusters x N rows).
// Exact alpha partial sums are left in s4c (kMaxClusters) for an optional M-shard allreduce.
int launch_select_local(cudaStream_t st, const double* W64, const double* alpha_old, const uint8_t* state,
                        const int* iters, int L_local, int64_t id_base, int N, uint32_t flags,
                        const float* X, int64_t ld, int64_t M_local, int* cluster, int* pc, int* qc,
                        int* csize, double* ups_max, int* counts, double* part, int nblk, double* s4c,
                        const int* nconv_g = nullptr);
// *out = converged candidates on this rank (L-shard: all-reduced into nconv_g of select_local)
int launch_count_converged(cudaStream_t st, const uint8_t* state, int L, int* out);
// nonfinite (device, may be null): this rank's count of rows retired by a non-finite update.
// sum_active < 0: take sum_active and n_iter (= t - 1) from the device iteration state ctl.
int launch_select_finish(cudaStream_t st, const double* W64, const int* iters, const int* counts,
                         const int* pc, const int* qc, const int* csize, const double* s4c,
                         int64_t id_base, int N, double M_global, uint32_t flags, int64_t sum_active,
                         int n_iter, const int* nonfinite, const IterCtl* ctl, RankSummary* summary, double* wsum);
// Merge all ranks' summaries (world x RankSummary, world x kMaxClusters x N), append the winner to
// Wacc row k, write the record.
int launch_merge_accept(cudaStream_t st, const RankSummary* all, const double* wall, int world, int N,
                        int i, double M_global, uint32_t flags, double* Wacc, int k, ComponentRecord* rec,
                        double* w_out);

// ---- fused tensor-core step (k_step_tc.cu)
// The fp16 X plane holds x * 2^-6 and the operand rows 2^4 w, so the GEMM1 accumulator is y / 4
// and its cube is directly the fp16 GEMM2 operand y^3 2^-6 (two multiplies per element); G is
// unscaled (x 2^12, exact) at the slot flush.  |x| < 2^-8 becomes fp16-subnormal (absolute
// error <= 2^-19 in x units, below the normal rounding of |x| ~ 2^-8).
constexpr float kXScale = 0x1.0p-6f;
struct TcPlan;
bool tc_supported(int N);
int tc_np(int N);
// Rows [0, n_coarse) are coarse (GEMM1 on W_hi), the rest fine (W_hi + W_lo).  Gp[s][a][n] fp32.
// L_act / n_coarse size the grid; when cnt (device [L_act, n_coarse]) is given they are upper
// bounds and the kernel takes the true values from cnt (tiles beyond exit at once).
// lo_capable: launch the LO-capable layout even if n_coarse == L_act (fine rows may appear).
// Slot range of one step launch: [s_base, s_base + s_count).  The whole step is one launch over
// all S slots; while a pipelined host upload is in flight the first step is launched piece by
// piece (each launch after its piece's copy event), which gives bitwise the same slot partials.
// Split-slot output of the tensor-core step (see SlotPartials): enable = 0 forces P = 1.
struct SplitOut {
  float* sub;
  int64_t sub_cap;
  const int* cnt_g;   // global active count (device; null: the host L_act)
  int enable;
};
struct Upload {
  int s_base;
  int s_count;
  int cl = 0;   // cluster size override (0: the default for NP)
};
// xshift (device, one int8 per 384-sample block of the local samples, launch_block_shift): the
// fp16 range shift of the GEMM2 operand; null: no shift.
// act (device): position a uses operand rows Whi / Wlo [act[a]] (by candidate id).
int launch_step_tc(cudaStream_t st, const __half* Xh, int64_t ldx, int64_t M, int NP, const __half* Whi,
                   const __half* Wlo, const int* act, int n_coarse, int L_act, int64_t slot_len, int S, float* Gp,
                   int64_t cap, const int* cnt, bool lo_capable, const Upload& up, const SplitOut& so,
                   const int8_t* xshift);
// fp16 range of the tensor-core step (DESIGN.md §5 "range"): for every 384-sample block b of the
// samples [m_lo, m_hi) (m_lo a multiple of 384), xshift[b] = the least dsh in [0, kMaxShift] with
// 1.01 max ||x_m||_2 <= 2^(7 + dsh).  The y^3 operand is scaled by 2^(-3 dsh) before its fp16
// rounding and G unscaled at the flush, so y^3 2^-6 2^(-3 dsh) < 2^15 < 65504 for |y| <= ||x_m||.
constexpr int kShiftBlock = 384;
constexpr int kMaxShift = 30;
int launch_block_shift(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, int64_t m_lo, int64_t m_hi,
                       int8_t* xshift);
// fp16 plane columns [m_lo, m_hi) (m_hi < 0: ldx); multiples of 8.
int launch_x_prepare_f16(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, int NP,
                         int64_t ldx, __half* Xh, int64_t m_lo = 0, int64_t m_hi = -1);


// ---- §3.3 reduction of X (k_reduce.cu)
// X~ = G X (Gf: d x N fp32 rows) into Xr (d x M, stride ldr) and, if Xh != null, the fp16 plane
// Xh [NPd][ldx] (rows >= d and columns >= M zero).
int launch_reduce_apply(cudaStream_t st, const float* Gf, int d, int N, const float* X, int64_t ld, int64_t M,
                        float* Xr, int64_t ldr, __half* Xh, int NPd, int64_t ldx);
// Candidates of component i in the reduced basis: W64 row j = G r_j / ||G r_j|| (d entries).
int launch_cand_basis(cudaStream_t st, uint64_t seed, int i, int64_t id_base, int64_t L_local, int N,
                      const double* G, int d, double* W64, uint8_t* state, uint8_t* keep, uint8_t* fine,
                      uint8_t fine_init, double* dprev);

// ---- boundary: whitening (k_whiten.cu)
int launch_row_mean(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, double* mean);
int launch_covariance(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, const double* mean,
                      double* part, int nsplit, double* C);
int launch_apply_whitening(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, const double* mean,
                           const double* V, float* Xw, int64_t ldo);

}  // namespace oica
