// Host runtime and C-ABI of liboica.so: context, memory planner, per-component driver loop,
// NCCL exchange, whitening eigensolver.  Kernels live in k_*.cu (launch wrappers in kernels.cuh).
#include <nvtx3/nvToolsExt.h>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/oica.h"
#include "common.cuh"
#include "kernels.cuh"
#include "merge.hpp"
#include "nccl_dl.hpp"

using namespace oica;

namespace {

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t k) {
    if (k <= n) return;
    release();
    if (k == 0) return;
    OICA_CUDA(cudaMalloc(&p, k * sizeof(T)));
    n = k;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

// Split-M slot policy: S depends only on M, so per-row results are identical
// for any GPU count in L-shard mode and any active-set size.
constexpr int64_t kSlotTarget = 65536;  // samples per slot (target) ...
constexpr int64_t kSlotMin = 128;       // ... but up to 30 slots of >= this many samples
constexpr int kMinSlots = 30;
constexpr int kMaxSlots = 128;
constexpr int kFlush = 4096;            // fp32 -> fp64 flush period (samples)
constexpr int64_t kSlotAlign = 384;       // multiple of every TC chunk width (64, 128, 192 samples)
constexpr int64_t kTcMinSamples = 16384;    // OICA_PREC_AUTO switches to tensor cores at this M
constexpr int64_t kSimtShortM = 65536;      // FP32 contexts below this M use short slots (plan_slots_for)
constexpr double kPromoteD = 1e-6;          // TC precision promotion: stagnating d below this ...
constexpr double kPromoteRatio = 0.3;       // ... (d > this * d_prev: stagnating) ...
constexpr int kPromoteT = 40;               // ... or t >= this
constexpr int kBatchRows = 2048;            // below this many active rows, iterations are enqueued ...
constexpr int kBatch = 8;                   // ... this many at a time without a host round trip
constexpr int kLoopUnroll = 4;             // iterations per WHILE-body execution (device-side loop)
constexpr double kBatchMaxWork = 1e8;       // ... when M x NP is below this (cfg 2: 1.6e7, cfg 3: 1.3e8)
constexpr int kHybridRowsPerRank = 128;     // OICA_SHARD_HYBRID: tail once global L_act <= this x world
constexpr int kTailMaxSlots = 1024;

}  // namespace

#ifdef OICA_EXPERIMENTS
// Driver entry points for green contexts (SM partitions), resolved at run time.
struct GreenApi {
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetDevResource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*SmResourceSplitByCount)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                                     unsigned) = nullptr;
  CUresult (*ResourceGenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
  CUresult (*GreenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*GreenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
  CUresult (*CtxFromGreenCtx)(CUcontext*, CUgreenCtx) = nullptr;
  CUresult (*CtxGetCurrent)(CUcontext*) = nullptr;
  CUresult (*CtxSetCurrent)(CUcontext) = nullptr;
  CUresult (*GreenCtxDestroy)(CUgreenCtx) = nullptr;
  CUresult (*StreamDestroy)(CUstream) = nullptr;
  bool ok = false;
  static GreenApi& get() {
    static GreenApi a = [] {
      GreenApi g;
      auto sym = [](const char* n) -> void* {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        return (cudaGetDriverEntryPoint(n, &p, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess) ? p : nullptr;
      };
      g.DeviceGet = (decltype(g.DeviceGet))sym("cuDeviceGet");
      g.DeviceGetDevResource = (decltype(g.DeviceGetDevResource))sym("cuDeviceGetDevResource");
      g.SmResourceSplitByCount = (decltype(g.SmResourceSplitByCount))sym("cuDevSmResourceSplitByCount");
      g.ResourceGenerateDesc = (decltype(g.ResourceGenerateDesc))sym("cuDevResourceGenerateDesc");
      g.GreenCtxCreate = (decltype(g.GreenCtxCreate))sym("cuGreenCtxCreate");
      g.GreenCtxStreamCreate = (decltype(g.GreenCtxStreamCreate))sym("cuGreenCtxStreamCreate");
      g.CtxFromGreenCtx = (decltype(g.CtxFromGreenCtx))sym("cuCtxFromGreenCtx");
      g.CtxGetCurrent = (decltype(g.CtxGetCurrent))sym("cuCtxGetCurrent");
      g.CtxSetCurrent = (decltype(g.CtxSetCurrent))sym("cuCtxSetCurrent");
      g.GreenCtxDestroy = (decltype(g.GreenCtxDestroy))sym("cuGreenCtxDestroy");
      g.StreamDestroy = (decltype(g.StreamDestroy))sym("cuStreamDestroy");
      g.ok = g.DeviceGet && g.DeviceGetDevResource && g.SmResourceSplitByCount && g.ResourceGenerateDesc &&
             g.GreenCtxCreate && g.GreenCtxStreamCreate && g.CtxFromGreenCtx && g.CtxGetCurrent && g.CtxSetCurrent &&
             g.GreenCtxDestroy && g.StreamDestroy;
      return g;
    }();
    return a;
  }
};

// Green-context split of the SMs for the NP = 256 step: partition A (128 SMs)
// runs 4-CTA multicast clusters, partition B (the other 20) 2-CTA clusters, concurrently.
struct GreenSplit {
  bool tried = false, ok = false;
  CUgreenCtx gA = nullptr, gB = nullptr;
  CUcontext cA = nullptr, cB = nullptr;
  CUstream sA = nullptr, sB = nullptr;
  cudaEvent_t fork = nullptr, jA = nullptr, jB = nullptr;
  unsigned smA = 0, smB = 0;
};

#endif

struct oica_ctx {
  oica_config cfg{};
  cudaStream_t st = nullptr;
  bool own_stream = false;
  std::string err;
  int num_sms = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  // data
  const float* X = nullptr;
  DevBuf<float> Xown;
  // pipelined host upload (oica_set_data_host): copy + fp16 conversion on a second stream, piece
  // by piece; the tensor-core step of the first iteration waits per piece (DESIGN.md §7 e2e)
  cudaStream_t cst = nullptr;
#ifdef OICA_EXPERIMENTS
  cudaStream_t st2 = nullptr;   // second launch of the mixed-cluster step (run_step)
  GreenSplit green;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
#endif
  cudaEvent_t x_ready_ev = nullptr, st_ev = nullptr;
  std::vector<cudaEvent_t> piece_ev;   // piece p of the upload is on the device (and converted)
  int pieces = 0;
  bool x_pending = false;
  int64_t piece_len = 0;
  int64_t N = 0, NP = 0, M = 0, ld = 0, Mg = 0;
  int precision = OICA_PREC_FP32;
  DevBuf<__half> Xh;   // TC operand plane
  int64_t ldx = 0;
  DevBuf<int8_t> xshift;   // fp16 range shift per 384-sample block (launch_block_shift)
  DevBuf<int> nonfinite;   // rows retired by a non-finite update in the current component
  DevBuf<int> nconv;       // converged count summed over ranks (L-shard selection, reading A4)
  DevBuf<IterCtl> ctl;     // device iteration state (t, k, update tickets): kernels/kernels.cuh
  // device-side do-while (CUDA graph with a WHILE node, DESIGN.md §5 "iteration"), rebuilt when a
  // parameter baked into its kernels changes
  struct LoopKey {   // every value a captured kernel parameter depends on (buffers by address)
    const void* X;
    const void* Xh;
    const void* buf[12];
    int64_t M, Mg, slot_len, ldx, vld;
    int vN, vNP, S, L_ub, K, precision;
    double tol;
    bool operator==(const LoopKey& o) const { return std::memcmp(this, &o, sizeof(LoopKey)) == 0; }
  };
  struct LoopGraph {
    bool valid = false;
    LoopKey key{};
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    std::vector<int> tiers;   // grid-size tiers (rows) of the WHILE nodes, in order
    int unroll = 1;           // iterations per body execution
    void reset() {
      if (x) cudaGraphExecDestroy(x);
      if (g) cudaGraphDestroy(g);
      x = nullptr;
      g = nullptr;
      valid = false;
    }
  } loop;
  // device-side loop timing, one pair per component slot (two components in flight, extract_impl)
  cudaEvent_t loop_ev0[2] = {nullptr, nullptr}, loop_ev1[2] = {nullptr, nullptr};
  int slot = 0;   // the component slot being enqueued
  cudaEvent_t comp_ev[2] = {nullptr, nullptr};   // a component slot's record copied to the host
  bool loop_persistent = false;   // the last device-side loop was the persistent FP32 kernel
  // pinned read-back of a component's results (one host wait per component on the fast path):
  // [ComponentRecord | IterCtl | w (256 doubles) | hist (2 (K + 1) ints)]
  char* pin = nullptr;
  size_t pin_bytes = 0;
  // two slots: the next component is enqueued before the host reads this one's record
  size_t pin_slot = 0;
  void ensure_pin(int K) {
    pin_slot = round_up(sizeof(ComponentRecord) + sizeof(IterCtl) + 256 * sizeof(double) + 2 * ((size_t)K + 1) * sizeof(int), 256);
    const size_t need = 2 * pin_slot;
    if (need <= pin_bytes) return;
    if (pin) cudaFreeHost(pin);
    pin = nullptr;
    pin_bytes = 0;
    OICA_CUDA(cudaHostAlloc((void**)&pin, need, cudaHostAllocDefault));
    pin_bytes = need;
  }
  char* pin_at(int j) { return pin + (size_t)j * pin_slot; }
  ComponentRecord* pin_rec(int j) { return (ComponentRecord*)pin_at(j); }
  IterCtl* pin_ctl(int j) { return (IterCtl*)(pin_at(j) + sizeof(ComponentRecord)); }
  double* pin_w(int j) { return (double*)(pin_at(j) + sizeof(ComponentRecord) + sizeof(IterCtl)); }
  int* pin_hist(int j) { return (int*)(pin_at(j) + sizeof(ComponentRecord) + sizeof(IterCtl) + 256 * sizeof(double)); }
  // the data the current component iterates on (DESIGN.md §5 "reduced X"): the full whitened X,
  // or X~ = G X in the d = N-k dimensional complement of the accepted rows (OICA_REDUCE_X)
  const float* vX = nullptr;
  int64_t vld = 0;
  const __half* vXh = nullptr;
  int vN = 0, vNP = 0;
  bool reduced = false;
  DevBuf<float> Xr, Gf;
  DevBuf<__half> Xrh;
  DevBuf<double> Gdev, Wacc_scratch;
  std::vector<double> Gh;   // host basis, d x N (rows orthonormal, orthogonal to W_acc)
  std::vector<double> Gh_last;   // basis of the last extracted component if it ran reduced
  int last_vN = 0;
  bool tc_ready = false;
  // slots
  int S = 1;
  int64_t slot_len = 0;
  // candidates
  bool have_cand = false;
  uint64_t seed = 0;
  int64_t L = 0, Ll = 0, id_base = 0;
  DevBuf<double> W64, alpha_old, Gp, s4p, Gsum, s4sum;
  DevBuf<float> Gp32;   // TC slot partials
  DevBuf<float> Gsub;   // TC split-slot parts (few active rows, common.cuh split_parts)
  int64_t sub_cap = 0;
  DevBuf<int> Lg;       // global active count (lock-step L-shard: all-reduced every iteration)
  DevBuf<double> Gfin, s4fin;   // final-w forward pass of the runs active at the cap
  DevBuf<float> W32;
  DevBuf<__half> Whi, Wlo;
  DevBuf<int> act0, act1, iters, Lact_dev, hist;
  DevBuf<int64_t> arghash;
  DevBuf<uint8_t> state, keep, fine;
  DevBuf<double> dprev;
  int* Lact_host = nullptr;   // mapped: [L_act, n_coarse]
  DevBuf<double> Wacc;
  // selection
  DevBuf<int> cluster, pc, qc, csize, counts;
  DevBuf<double> ups_max, part, s4c, wsum, wsum_all, w_out;
  DevBuf<RankSummary> summary, summary_all;
  DevBuf<ComponentRecord> rec;
  int nblk_alpha = 0;
  bool last_valid = false;
  // whitening scratch
  DevBuf<double> wh_mean, wh_part, wh_C, wh_V;
  // hybrid L -> M tail (OICA_SHARD_HYBRID): the gathered runs, identical on all ranks
  struct Tail {
    DevBuf<double> pack, pack_all, dense, W64, alpha, dprev, Gsum, s4sum, Gp, s4p;
    DevBuf<float> Gp32, W32;
    DevBuf<__half> Whi, Wlo;
    DevBuf<int64_t> ids;
    DevBuf<int> iters, act0, act1, hist, cnt_all;
    DevBuf<uint8_t> state, keep, fine;
  } tail;

  // stats
  oica_stats stats{};
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;

  // NCCL failure handling: with a communicator every host wait polls the stream and
  // NCCL's asynchronous error state, and gives up after nccl_timeout_s (OICA_NCCL_TIMEOUT_S,
  // default 900 s): a peer that died or never joined cannot hang the caller.  The communicator is
  // then aborted and the context is usable only for oica_destroy (`broken`).
  bool broken = false;
  double nccl_timeout_s = 900.0;
  void abort_comm(const std::string& why) {
    if (comm) Nccl::get().CommAbort(comm);
    comm = nullptr;
    broken = true;
    throw Error(OICA_ERR_NCCL, why);
  }
  void wait() {
    if (!comm) {
      OICA_CUDA(cudaStreamSynchronize(st));
      return;
    }
    auto& nc = Nccl::get();
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t spin = 0;; ++spin) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) return;
      if (q != cudaErrorNotReady) OICA_CUDA(q);
      if ((spin & 255) == 0) {
        ncclResult_t ae = ncclSuccess;
        nc.CommGetAsyncError(comm, &ae);
        if (ae != ncclSuccess && ae != ncclInProgress)
          abort_comm(std::string("NCCL asynchronous error: ") + nc.GetErrorString(ae));
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > nccl_timeout_s)
          abort_comm("collective wait exceeded " + std::to_string((int)nccl_timeout_s) +
                     " s (OICA_NCCL_TIMEOUT_S): a peer rank stopped or never called");
      }
      if (spin > 64) std::this_thread::yield();
    }
  }
  // CUDA-event time of the NCCL exchanges inside extract (oica_stats.exchange_ms)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> xev;
  size_t xev_used = 0;
  template <class F>
  void exchange(F&& f) {
    if (xev_used == xev.size()) {
      cudaEvent_t a, b;
      OICA_CUDA(cudaEventCreate(&a));
      OICA_CUDA(cudaEventCreate(&b));
      xev.emplace_back(a, b);
    }
    auto& e = xev[xev_used++];
    OICA_CUDA(cudaEventRecord(e.first, st));
    f();
    OICA_CUDA(cudaEventRecord(e.second, st));
    ++stats.exchange_calls;
  }

  int world() const { return cfg.world; }
  bool tc() const { return precision == OICA_PREC_TC || precision == OICA_PREC_TC_SPLIT; }
  bool split() const { return precision == OICA_PREC_TC_SPLIT; }
  // slot partials of the last step; cnt_g / L_g: the global active count that chose its split
  // parts (device pointer, or the host value when null)
  SlotPartials partials(const int* cnt_g, int L_g) const {
    return tc() ? SlotPartials{Gp32.p, true, Gsub.p, sub_cap, cnt_g, L_g} : SlotPartials{Gp.p, false};
  }
  EvalPoint eval_point() const {
    return tc() ? EvalPoint{Whi.p, Wlo.p, nullptr, vNP} : EvalPoint{nullptr, nullptr, W32.p, vNP};
  }
  Promotion promotion() const {
#ifdef OICA_EXPERIMENTS
    static const double pd = getenv("OICA_PROMOTE_D") ? atof(getenv("OICA_PROMOTE_D")) : kPromoteD;
    static const double pr = getenv("OICA_PROMOTE_RATIO") ? atof(getenv("OICA_PROMOTE_RATIO")) : kPromoteRatio;
    static const int pt = getenv("OICA_PROMOTE_T") ? atoi(getenv("OICA_PROMOTE_T")) : kPromoteT;
#else
    constexpr double pd = kPromoteD, pr = kPromoteRatio;
    constexpr int pt = kPromoteT;
#endif
    Promotion p = tc() ? Promotion{fine.p, dprev.p, pd, pr, pt} : Promotion{nullptr, nullptr, 0.0, 0.0, 0};
    p.nonfinite = nonfinite.p;
    return p;
  }
  const uint8_t* fine_flags() const { return tc() ? fine.p : nullptr; }
  // a communicator exists for world > 1, or at world == 1 when a unique id is passed (the
  // exchange / allreduce code paths then run over one rank: tests on a single GPU)
  bool mshard() const { return comm && cfg.shard_mode == OICA_SHARD_M; }
  bool hybrid() const { return comm && cfg.shard_mode == OICA_SHARD_HYBRID; }
  bool collective() const { return comm != nullptr; }

  void count(int n) { stats.kernel_launches += n; }
  cudaEvent_t event() {
    if (ev_used == ev.size()) {
      cudaEvent_t e;
      OICA_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
    return ev[ev_used++];
  }
  // per-iteration log (oica_get_iteration_log): the iteration each timed event pair belongs to
  int cur_t = 0;
  std::vector<int> ev_t;
  std::vector<std::pair<int, float>> pairs;   // (iteration, ms) of the last harvest
  std::vector<oica_iteration_record> iter_log;
  void mark_pair() { ev_t.push_back(cur_t); }
  void harvest_events() {
    wait();
    for (size_t k = 0; k < xev_used; ++k) {
      float ms = 0.f;
      OICA_CUDA(cudaEventElapsedTime(&ms, xev[k].first, xev[k].second));
      stats.exchange_ms += ms;
    }
    xev_used = 0;
    pairs.clear();
    for (size_t k = 0; k + 1 < ev_used; k += 2) {
      float ms = 0.f;
      OICA_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
      stats.step_ms += ms;
      pairs.emplace_back(k / 2 < ev_t.size() ? ev_t[k / 2] : 0, ms);
    }
    ev_used = 0;
    ev_t.clear();
  }
};

namespace {

oica_status fail(oica_ctx* ctx, oica_status s, const std::string& m) {
  if (ctx) ctx->err = m;
  return s;
}

template <class F>
oica_status guard(oica_ctx* ctx, F&& f) {
  try {
    if (ctx) {
      ctx->err.clear();
      OICA_REQUIRE(!ctx->broken, OICA_ERR_NCCL, "context unusable after an NCCL failure: destroy it");
      OICA_CUDA(cudaSetDevice(ctx->cfg.device));
    }
    f();
    return OICA_OK;
  } catch (const Error& e) {
    return fail(ctx, e.status, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ctx, OICA_ERR_OUT_OF_MEMORY, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, OICA_ERR_CUDA, e.what());
  }
}

// Cyclic Jacobi eigensolver for a symmetric N x N matrix (row-major, fp64).
void jacobi_eigh(std::vector<double>& A, int n, std::vector<double>& d, std::vector<double>& E) {
  E.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) E[(size_t)i * n + i] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[(size_t)i * n + j]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += a(i, j) * a(i, j);
        if (i != j) off += a(i, j) * a(i, j);
      }
    if (off <= 1e-30 * tot) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = a(p, q);
        if (std::fabs(apq) < 1e-300) continue;
        double app = a(p, p), aqq = a(q, q);
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          double ekp = E[(size_t)k * n + p], ekq = E[(size_t)k * n + q];
          E[(size_t)k * n + p] = c * ekp - s * ekq;
          E[(size_t)k * n + q] = s * ekp + c * ekq;
        }
      }
  }
  d.resize(n);
  for (int i = 0; i < n; ++i) d[i] = a(i, i);
}

// Split-M slot plan: slot length is a function of the GLOBAL M only (determinism across GPU
// counts, tilings and active-set sizes); the local slot count follows from the local M.
void plan_slots_for(int64_t M_global, int64_t M_local, bool fp32, int64_t* slot_len, int* S_local) {
  if (fp32 && M_global < kSimtShortM) {
    // FP32 step at small M (the paper's own experiments, M = 1e4): one CTA per (64-row tile, slot)
    // streams its slot chunk by chunk, so short slots (>= 128 samples, up to 128 of them, 64-aligned
    // = the FP32 chunk) give the few row tiles enough CTAs: a 1e4-sample step 23 -> 12 us.  (One
    // 64-sample chunk per slot, up to 256 slots, measured slower: a unit's fixed latencies dominate
    // and the update then sums twice the partials.)
    const int64_t S = std::max<int64_t>(1, std::min<int64_t>(kMaxSlots, ceil_div(M_global, 128)));
    *slot_len = round_up(ceil_div(M_global, S), 64);
    *S_local = std::max(1, (int)ceil_div(M_local, *slot_len));
    return;
  }
  // one CTA per (row tile, slot): long slots amortise each CTA's set-up (TMEM allocation, W
  // load, pipeline fill, G flush: ~13% of the step at 8192-sample slots and N = 128), while up
  // to 30 slots (of >= 128 samples) keep enough CTAs per row tile for small L and small M
#ifdef OICA_EXPERIMENTS
  static int64_t target = [] { const char* e = getenv("OICA_SLOT_TARGET"); return e ? atoll(e) : kSlotTarget; }();
  static int64_t min_slots = [] { const char* e = getenv("OICA_MIN_SLOTS"); return e ? atoll(e) : (int64_t)kMinSlots; }();
#else
  constexpr int64_t target = kSlotTarget, min_slots = kMinSlots;
#endif
  int64_t S = std::max<int64_t>(std::min<int64_t>(min_slots, M_global / kSlotMin), M_global / target);
  S = std::max<int64_t>(1, std::min<int64_t>(kMaxSlots, S));
  *slot_len = round_up(ceil_div(M_global, S), kSlotAlign);
  *S_local = std::max(1, (int)ceil_div(M_local, *slot_len));
}

void plan_slots(oica_ctx* c) { plan_slots_for(c->Mg, c->M, !c->tc(), &c->slot_len, &c->S); }

void ensure_candidate_buffers(oica_ctx* c) {
  size_t Ll = (size_t)c->Ll, N = (size_t)c->N, NP = (size_t)c->NP;
  c->nonfinite.ensure(1);
  c->nconv.ensure(1);
  c->ctl.ensure(1);
  c->W64.ensure(Ll * N);
  c->alpha_old.ensure(Ll);
  c->iters.ensure(Ll);
  c->state.ensure(Ll);
  c->keep.ensure(Ll);
  c->act0.ensure(Ll);
  c->act1.ensure(Ll);
  c->Lact_dev.ensure(4);   // [L_act, n_coarse] + the unrolled loop body's gate (2)
  c->Lg.ensure(1);
  c->fine.ensure(Ll);
  c->dprev.ensure(Ll);
  if (c->tc()) {
    c->Gp32.ensure((size_t)c->S * Ll * NP);
    // split parts exist only while round_up(tiles, 2) S <= kSplitTarget / 2 (split_parts)
    c->sub_cap = std::min<int64_t>(round_up((int64_t)Ll, 128), 128 * std::max(1, kSplitTarget / 2 / c->S));
    c->Gsub.ensure((size_t)c->S * kSplitMax * c->sub_cap * NP);
    c->Whi.ensure(Ll * NP);
    c->Wlo.ensure(Ll * NP);
  } else {
    c->Gp.ensure((size_t)c->S * Ll * NP);
    c->s4p.ensure((size_t)c->S * Ll);
    c->W32.ensure(Ll * NP);
  }
  if (c->mshard()) {
    c->Gsum.ensure(Ll * NP);
    c->s4sum.ensure(Ll);
  }
  c->cluster.ensure(Ll);
  c->pc.ensure(kMaxClusters);
  c->qc.ensure(kMaxClusters);
  c->csize.ensure(kMaxClusters);
  c->counts.ensure(4);
  c->ups_max.ensure(1);
  // exact-alpha blocks: enough in flight to stream X at HBM rate (>= ~512 samples per block)
  c->nblk_alpha = (int)std::max<int64_t>(1, std::min<int64_t>(8 * c->num_sms, ceil_div(c->M, 512)));
  c->part.ensure((size_t)kMaxClusters * c->nblk_alpha);
  c->s4c.ensure(kMaxClusters);
  c->wsum.ensure(kMaxClusters * N);
  c->wsum_all.ensure((size_t)c->cfg.world * kMaxClusters * N);
  c->summary.ensure(1);
  c->summary_all.ensure((size_t)c->cfg.world);
  c->rec.ensure(1);
  c->w_out.ensure(N);
  c->Wacc.ensure(N * N);
}

// Every consumer of the data other than the first tensor-core step orders itself after a
// pending pipelined upload.
void sync_x(oica_ctx* c) {
  if (!c->x_pending) return;
  OICA_CUDA(cudaStreamWaitEvent(c->st, c->x_ready_ev, 0));
  c->x_pending = false;
}


// Step-kernel operand rows of candidates 0..L-1 (by id) from the fp64 master; afterwards the
// fused update keeps the rows of the active candidates current.
void build_operand(oica_ctx* c, int L) {
  if (c->tc())
    c->count(launch_operand_f16x2(c->st, L, c->W64.p, c->vN, c->vNP, c->fine.p, c->Whi.p, c->Wlo.p));
  else
    c->count(launch_operand_f32(c->st, L, c->W64.p, c->vN, c->vNP, c->W32.p));
}

// The fused update of one iteration (K3 + K4, kernels.cuh launch_update) over the L_ub (upper
// bound) active positions of act_in, compacting into act_out.
UpdateArgs update_args(oica_ctx* c, SlotPartials G, const double* s4, int S, int64_t cap, const int* act_in,
                       int* act_out, int L_ub, double tol, int* hist) {
  UpdateArgs u{};
  u.G = G;
  u.s4p = s4;
  u.S = S;
  u.cap = cap;
  u.ldg = c->vNP;
  u.ev = c->eval_point();
  u.act_in = act_in;
  u.act_out = act_out;
  u.copy_back = 0;
  u.L_ub = L_ub;
  u.cnt_in = c->Lact_dev.p;
  u.cnt_out = c->Lact_dev.p;
  u.host_mapped = c->Lact_host;
  u.hist = hist;
  u.Wacc = c->Wacc.p;
  u.N = c->vN;
  u.M = (double)c->Mg;
  u.tol = tol;
  u.W64 = c->W64.p;
  u.alpha_old = c->alpha_old.p;
  u.iters = c->iters.p;
  u.state = c->state.p;
  u.keep = c->keep.p;
  u.pr = c->promotion();
  u.ctl = c->ctl.p;
  u.compact = 1;
  return u;
}

// the fused update, with the compaction inside for up to kUpdateCompactRows rows, else a 1024-thread
// compaction kernel after it (which then also ends the iteration)
void run_update(oica_ctx* c, UpdateArgs u) {
  u.compact = u.L_ub <= kUpdateCompactRows ? 1 : 0;
  c->count(launch_update(c->st, u, c->vNP));
  if (!u.compact) c->count(launch_compact_iter(c->st, u));
}

#ifdef OICA_EXPERIMENTS
// Lazily builds the green-context split; false (and never retried) if unavailable.
bool green_ready(oica_ctx* c) {
  GreenSplit& g = c->green;
  if (g.tried) return g.ok;
  g.tried = true;
  GreenApi& api = GreenApi::get();
  if (!api.ok) {
    if (getenv("OICA_TRACE")) fprintf(stderr, "[oica] green split unavailable: driver entry points\n");
    return false;
  }
  CUdevice dev;
  CUdevResource sm, grp[1], rem;
  unsigned nb = 1;
  static const int smA_env = [] { const char* e = getenv("OICA_GREEN_SMS"); return e ? atoi(e) : 128; }();
  auto fail_trace = [](const char* what) {
    if (getenv("OICA_TRACE")) fprintf(stderr, "[oica] green split unavailable: %s\n", what);
    return false;
  };
  if (api.DeviceGet(&dev, c->cfg.device) != CUDA_SUCCESS ||
      api.DeviceGetDevResource(dev, &sm, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      api.SmResourceSplitByCount(grp, &nb, &sm, &rem, 0, (unsigned)smA_env) != CUDA_SUCCESS || nb != 1 ||
      rem.sm.smCount < 2)
    return fail_trace("SM split");
  CUdevResourceDesc dA, dB;
  if (api.ResourceGenerateDesc(&dA, &grp[0], 1) != CUDA_SUCCESS || api.ResourceGenerateDesc(&dB, &rem, 1) != CUDA_SUCCESS ||
      api.GreenCtxCreate(&g.gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      api.GreenCtxCreate(&g.gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      api.GreenCtxStreamCreate(&g.sA, g.gA, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      api.GreenCtxStreamCreate(&g.sB, g.gB, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      api.CtxFromGreenCtx(&g.cA, g.gA) != CUDA_SUCCESS || api.CtxFromGreenCtx(&g.cB, g.gB) != CUDA_SUCCESS)
    return fail_trace("green context");
  OICA_CUDA(cudaEventCreateWithFlags(&g.fork, cudaEventDisableTiming));
  OICA_CUDA(cudaEventCreateWithFlags(&g.jA, cudaEventDisableTiming));
  OICA_CUDA(cudaEventCreateWithFlags(&g.jB, cudaEventDisableTiming));
  g.smA = grp[0].sm.smCount;
  g.smB = rem.sm.smCount;
  g.ok = true;
  if (getenv("OICA_TRACE")) fprintf(stderr, "[oica] green split: %u + %u SMs\n", g.smA, g.smB);
  return true;
}

// The green split (an experiment, OICA_TC_GREEN=1): full-size NP = 256 steps.  Measured equal to
// 2-CTA clusters on all 148 SMs (same clock: the 4-CTA clusters' higher clock came from the 16 SMs
// they leave idle, not from the smaller L2 stream; profiles/r01/tc_experiments).
bool green_step(oica_ctx* c, int L_act) {
  static const bool on = [] { const char* e = getenv("OICA_TC_GREEN"); return e && atoi(e) == 1; }();
  static const bool cl_env = getenv("OICA_TC_CL") != nullptr;
  return on && !cl_env && c->vNP == 256 && c->S >= 10 && L_act >= 64 * 128 && green_ready(c);
}

// Mixed 4-/2-CTA cluster launches (run_step), an experiment (OICA_TC_MIXED=1; measured slower
// than 2-CTA clusters alone, profiles/r01/tc_experiments): NP = 256, >= 64 row tiles.
bool mixed_clusters(const oica_ctx* c, int L_act) {
  static const bool on = [] { const char* e = getenv("OICA_TC_MIXED"); return e && atoi(e) == 1; }();
  static const bool cl_env = getenv("OICA_TC_CL") != nullptr;
  return on && !cl_env && c->vNP == 256 && c->S >= 10 && L_act >= 64 * 128;
}

#endif

// One fused contraction over the active rows (positions 0..L_act-1; rows >= n_coarse are fine)
// into the slots.  With cnt (device [L_act, n_coarse]) the host values are upper bounds that
// only size the grid (iterations enqueued without a host round trip).
void run_step(oica_ctx* c, const int* act, int L_act, int n_coarse, const int* cnt, const int* cnt_g, bool lo_capable,
              bool timed, bool split = true) {
  const SplitOut so{c->Gsub.p, c->sub_cap, cnt_g, split ? 1 : 0};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    e0 = c->event();
    c->mark_pair();
    OICA_CUDA(cudaEventRecord(e0, c->st));
  }
  int n;
  if (c->tc() && c->x_pending && !c->reduced) {
    // pipelined host upload in flight: one launch per piece of whole slots, each after its
    // piece's copy + conversion (same slot partials as one launch over all slots)
    const int spp = (int)(c->piece_len / c->slot_len);
    n = 0;
    for (int p = 0; p < c->pieces; ++p) {
      OICA_CUDA(cudaStreamWaitEvent(c->st, c->piece_ev[p], 0));
      const int s0 = p * spp, s1 = std::min(c->S, s0 + spp);
      if (s1 > s0)
        n += launch_step_tc(c->st, c->vXh, c->ldx, c->M, c->vNP, c->Whi.p, c->Wlo.p, act, n_coarse, L_act, c->slot_len,
                            c->S, c->Gp32.p, c->Ll, cnt, lo_capable, Upload{s0, s1 - s0}, so, c->xshift.p);
    }
    sync_x(c);
#ifdef OICA_EXPERIMENTS
  } else if (c->tc() && green_step(c, L_act)) {
    // 4-CTA multicast clusters on a 128-SM partition (a quarter of the L2 -> SM stream: less power,
    // a higher clock; 4-CTA clusters alone fit on only 132 SMs) and 2-CTA clusters on the other
    // 20 SMs, concurrently, slots split in proportion.  Same arithmetic per slot.
    sync_x(c);
    GreenSplit& g = c->green;
    GreenApi& api = GreenApi::get();
    const int S_a = std::min(c->S - 1, std::max(1, (int)std::lround((double)c->S * g.smA / (g.smA + g.smB))));
    const int S_b = c->S - S_a;
    OICA_CUDA(cudaEventRecord(g.fork, c->st));
    OICA_CUDA(cudaStreamWaitEvent((cudaStream_t)g.sA, g.fork, 0));
    OICA_CUDA(cudaStreamWaitEvent((cudaStream_t)g.sB, g.fork, 0));
    struct CtxRestore {   // the calling thread leaves in its own context even if a launch throws
      GreenApi& api;
      CUcontext prev = nullptr;
      explicit CtxRestore(GreenApi& a) : api(a) { api.CtxGetCurrent(&prev); }
      ~CtxRestore() { api.CtxSetCurrent(prev); }
    } restore(api);
    api.CtxSetCurrent(g.cA);
    n = launch_step_tc((cudaStream_t)g.sA, c->vXh, c->ldx, c->M, c->vNP, c->Whi.p, c->Wlo.p, act, n_coarse, L_act,
                       c->slot_len, c->S, c->Gp32.p, c->Ll, cnt, lo_capable, Upload{0, S_a, 4}, so, c->xshift.p);
    api.CtxSetCurrent(g.cB);
    n += launch_step_tc((cudaStream_t)g.sB, c->vXh, c->ldx, c->M, c->vNP, c->Whi.p, c->Wlo.p, act, n_coarse, L_act,
                        c->slot_len, c->S, c->Gp32.p, c->Ll, cnt, lo_capable, Upload{S_a, S_b, 2}, so, c->xshift.p);
    OICA_CUDA(cudaEventRecord(g.jA, (cudaStream_t)g.sA));
    OICA_CUDA(cudaEventRecord(g.jB, (cudaStream_t)g.sB));
    OICA_CUDA(cudaStreamWaitEvent(c->st, g.jA, 0));
    OICA_CUDA(cudaStreamWaitEvent(c->st, g.jB, 0));
  } else if (c->tc() && mixed_clusters(c, L_act)) {
    // experiment: 4-CTA multicast clusters (a quarter of the L2 -> SM stream, less power, a higher
    // clock) fit on only 132 of the 148 SMs (cudaOccupancyMaxActiveClusters: 33 clusters); a
    // concurrent 2-CTA launch on a second stream takes the slots meant for the other 16 SMs.
    // Same arithmetic per slot.
    sync_x(c);
    static const int sms_b = [] { const char* e = getenv("OICA_TC_MIXED_SMS"); return e ? atoi(e) : 16; }();
    const int S_b = std::max(1, (int)((int64_t)c->S * sms_b / 148));
    const int S_a = c->S - S_b;
    if (!c->st2) {
      OICA_CUDA(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
      OICA_CUDA(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
      OICA_CUDA(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
    }
    OICA_CUDA(cudaEventRecord(c->fork_ev, c->st));
    OICA_CUDA(cudaStreamWaitEvent(c->st2, c->fork_ev, 0));
    n = launch_step_tc(c->st, c->vXh, c->ldx, c->M, c->vNP, c->Whi.p, c->Wlo.p, act, n_coarse, L_act, c->slot_len, c->S,
                       c->Gp32.p, c->Ll, cnt, lo_capable, Upload{0, S_a, 4}, so, c->xshift.p);
    n += launch_step_tc(c->st2, c->vXh, c->ldx, c->M, c->vNP, c->Whi.p, c->Wlo.p, act, n_coarse, L_act, c->slot_len, c->S,
                        c->Gp32.p, c->Ll, cnt, lo_capable, Upload{S_a, S_b, 2}, so, c->xshift.p);
    OICA_CUDA(cudaEventRecord(c->join_ev, c->st2));
    OICA_CUDA(cudaStreamWaitEvent(c->st, c->join_ev, 0));
#endif
  } else if (c->tc()) {
    sync_x(c);
    n = launch_step_tc(c->st, c->vXh, c->ldx, c->M, c->vNP, c->Whi.p, c->Wlo.p, act, n_coarse, L_act, c->slot_len,
                       c->S, c->Gp32.p, c->Ll, cnt, lo_capable, Upload{0, c->S}, so, c->xshift.p);
  } else {
    sync_x(c);
    n = launch_step_simt(c->st, c->vX, c->vld, c->M, c->vN, c->vNP, c->W32.p, act, L_act, c->slot_len, c->S, kFlush,
                         c->Gp.p, c->s4p.p, c->Ll, cnt);
  }
  OICA_CUDA(cudaGetLastError());
  c->count(n);
  c->stats.step_launches += n;
  if (timed) {
    e1 = c->event();
    OICA_CUDA(cudaEventRecord(e1, c->st));
  }
}

// Work counters of one executed iteration with L_act rows, n_coarse of them coarse.
void account_iteration(oica_ctx* c, int L_act, int n_coarse, int64_t M_work = -1, bool timed = true) {
  if (M_work < 0) M_work = c->M;
  if (!timed) {   // an iteration of the device-side loop: counted, its step not timed on its own
    c->stats.iterations += 1;
    c->stats.sum_active += L_act;
    c->stats.graph_iterations += 1;
    c->stats.graph_flops += (double)L_act * (4.0 * (double)c->vN * (double)c->Mg + 3.0 * (double)c->Mg) *
                            ((double)M_work / (double)c->Mg);
    if (c->tc()) c->stats.fine_rows += L_act - n_coarse;
    return;
  }
  double issued;
  if (c->tc()) {
    int64_t tiles = ceil_div(L_act, 128), lo_tiles = n_coarse < L_act ? tiles - n_coarse / 128 : 0;
    issued = 128.0 * (double)c->vNP * (double)M_work * 2.0 * (2.0 * (double)tiles + 2.0 * (double)lo_tiles);
    c->stats.fine_rows += L_act - n_coarse;
  } else {
    issued = (double)round_up(L_act, 64) * (double)c->vNP * (double)M_work * 4.0;
  }
  c->stats.iterations += 1;
  c->stats.sum_active += L_act;
  c->stats.step_flops += (double)L_act * (4.0 * (double)c->vN * (double)c->Mg + 3.0 * (double)c->Mg) *
                         ((double)M_work / (double)c->Mg);
  c->stats.step_issued_flops += issued;
}

void check_launch() { OICA_CUDA(cudaGetLastError()); }

// OICA_TRACE=1: per-component host wall-clock phases on stderr (development aid)
// Per-component phase trace: NVTX ranges (component i > a1 draw / a2-a6 iterate / a7 select /
// accept; no-ops unless a profiler is attached) and, with OICA_TRACE, host timings on stderr.
struct PhaseTrace {
  bool on = getenv("OICA_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  std::string line;
  int depth = 0;        // open NVTX ranges
  bool phases = true;   // phase ranges (false when components are enqueued one ahead: one range per
                        // component's enqueue)
  void push(const char* name) {
    nvtxRangePushA(name);
    ++depth;
  }
  void pop() {
    if (depth > 0) {
      nvtxRangePop();
      --depth;
    }
  }
  void begin(int i) {
    while (depth > 0) pop();
    push(("oica component " + std::to_string(i)).c_str());
    if (phases) push("a1 draw (P:237-239)");
  }
  void end() {
    while (depth > 0) pop();
  }
  ~PhaseTrace() {
    while (depth > 0) pop();
  }
  void mark(const char* what) {
    // `what` ended; the next phase's range opens
    if (phases) {
      const std::string w(what);
      pop();
      if (w == "init")
        push("a2-a6 iterate (P:241-256)");
      else if (w == "iterate")
        push("a7 select (P:257-259)");
      else if (w == "select")
        push("accept (P:264)");
    }
    if (!on) return;
    auto t1 = std::chrono::steady_clock::now();
    line += std::string(" ") + what + "=" +
            std::to_string(std::chrono::duration<double, std::micro>(t1 - t0).count()).substr(0, 7) + "us";
    t0 = t1;
  }
  // host time enqueueing iteration batches vs waiting for them (iterate phase)
  double enq_us = 0.0, wait_us = 0.0;
  int batches = 0;
  std::chrono::steady_clock::time_point tb;
  void batch_begin() {
    if (on) tb = std::chrono::steady_clock::now();
  }
  void batch_enqueued() {
    if (!on) return;
    auto t1 = std::chrono::steady_clock::now();
    enq_us += std::chrono::duration<double, std::micro>(t1 - tb).count();
    tb = t1;
  }
  void batch_done() {
    if (!on) return;
    wait_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tb).count();
    ++batches;
  }
  void flush(int i) {
    while (depth > 0) pop();
    if (on)
      fprintf(stderr, "[oica] component %d:%s (iterate: %d batches, enqueue %.0fus, wait %.0fus)\n", i, line.c_str(),
              batches, enq_us, wait_us);
    line.clear();
    enq_us = wait_us = 0.0;
    batches = 0;
  }
};

// ---- §3.3 reduction of X (Alg. 2 lines 4-12) ---------------------------
// The paper builds the complement basis as G = (F~F~^T)^{-1/2} F~ with F = I - W^T W.  Any
// orthonormal basis of the complement gives the same trajectories (w = G^T b; the update of
// eq. (5) is equivariant under b -> U b, X~ -> U X~ for orthogonal U; reading A9),
// so the runtime uses Householder reflections: O(N^2 k) once for a caller prefix, then one
// reflection per accepted row, O(d N), instead of a d x d inverse square root per component.

// Rows of G (N-k x N): the last N-k columns of Q in the Householder QR of W^T (W: k x N, rows
// orthonormal).
void complement_basis(const double* W, int k, int N, std::vector<double>& G) {
  std::vector<double> A((size_t)N * std::max(k, 1));   // A[n][j] = W[j][n]
  for (int j = 0; j < k; ++j)
    for (int n = 0; n < N; ++n) A[(size_t)n * k + j] = W[(size_t)j * N + n];
  std::vector<double> Q((size_t)N * N, 0.0), v(N), u(N);
  for (int n = 0; n < N; ++n) Q[(size_t)n * N + n] = 1.0;
  for (int j = 0; j < k; ++j) {
    double nx = 0.0;
    for (int r = j; r < N; ++r) nx += A[(size_t)r * k + j] * A[(size_t)r * k + j];
    nx = std::sqrt(nx);
    double a0 = A[(size_t)j * k + j];
    double alpha = a0 >= 0 ? -nx : nx;
    for (int r = j; r < N; ++r) v[r] = A[(size_t)r * k + j];
    v[j] -= alpha;
    double vn2 = 0.0;
    for (int r = j; r < N; ++r) vn2 += v[r] * v[r];
    if (vn2 <= 0.0) continue;
    for (int cidx = j; cidx < k; ++cidx) {   // A <- H A
      double sdot = 0.0;
      for (int r = j; r < N; ++r) sdot += v[r] * A[(size_t)r * k + cidx];
      sdot *= 2.0 / vn2;
      for (int r = j; r < N; ++r) A[(size_t)r * k + cidx] -= sdot * v[r];
    }
    for (int n = 0; n < N; ++n) {             // Q <- Q H
      double sdot = 0.0;
      for (int r = j; r < N; ++r) sdot += Q[(size_t)n * N + r] * v[r];
      sdot *= 2.0 / vn2;
      for (int r = j; r < N; ++r) Q[(size_t)n * N + r] -= sdot * v[r];
    }
  }
  int d = N - k;
  G.assign((size_t)d * N, 0.0);
  for (int r = 0; r < d; ++r)
    for (int n = 0; n < N; ++n) G[(size_t)r * N + n] = Q[(size_t)n * N + (k + r)];
}

// G (d x N) -> rows 2..d of H G, H the reflection taking the unit vector b (reduced coordinates of
// the accepted row) to -+e_1: the first row of H G is +-w, the rest span the new complement.
void deflate_basis(std::vector<double>& G, int d, int N, const double* b) {
  std::vector<double> v(b, b + d), u(N, 0.0);
  double nb = 0.0;
  for (int r = 0; r < d; ++r) nb += b[r] * b[r];
  nb = std::sqrt(nb);
  v[0] -= b[0] >= 0 ? -nb : nb;
  double vn2 = 0.0;
  for (int r = 0; r < d; ++r) vn2 += v[r] * v[r];
  if (vn2 > 0.0) {
    for (int r = 0; r < d; ++r)
      for (int n = 0; n < N; ++n) u[n] += v[r] * G[(size_t)r * N + n];
    for (int r = 0; r < d; ++r) {
      double f = 2.0 * v[r] / vn2;
      for (int n = 0; n < N; ++n) G[(size_t)r * N + n] -= f * u[n];
    }
  }
  G.erase(G.begin(), G.begin() + N);
}

int simt_np(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256; }

void use_full_view(oica_ctx* c) {
  c->vX = c->X;
  c->vld = c->ld;
  c->vXh = c->Xh.p;
  c->vN = (int)c->N;
  c->vNP = (int)c->NP;
  c->reduced = false;
}

// X~ = G X for the current host basis c->Gh (d = rows): fp32 copy (selection, FP32 step) and the
// fp16 tensor-core plane.
void use_reduced_view(oica_ctx* c, int d) {
  const int N = (int)c->N;
  sync_x(c);
  c->Gdev.ensure((size_t)d * N);
  c->Gf.ensure((size_t)d * N);
  std::vector<float> gf(c->Gh.begin(), c->Gh.begin() + (size_t)d * N);
  OICA_CUDA(cudaMemcpyAsync(c->Gdev.p, c->Gh.data(), sizeof(double) * d * N, cudaMemcpyHostToDevice, c->st));
  OICA_CUDA(cudaMemcpyAsync(c->Gf.p, gf.data(), sizeof(float) * d * N, cudaMemcpyHostToDevice, c->st));
  c->Xr.ensure((size_t)N * c->M);
  int npd = c->tc() ? tc_np(d) : simt_np(d);
  if (c->tc()) c->Xrh.ensure((size_t)c->NP * c->ldx);
  c->count(launch_reduce_apply(c->st, c->Gf.p, d, N, c->X, c->ld, c->M, c->Xr.p, c->M, c->tc() ? c->Xrh.p : nullptr,
                               npd, c->ldx));
  check_launch();
  c->wait();   // gf is a host temporary
  c->vX = c->Xr.p;
  c->vld = c->M;
  c->vXh = c->tc() ? c->Xrh.p : nullptr;
  c->vN = d;
  c->vNP = npd;
  c->reduced = true;
}

// alpha_old of the L_fin runs still active (positions act[0..L_fin), count in Lact_dev) at their
// final w: one step over those rows, s4 = w_e . G (TC identity) or the SIMT s4 partials.
void refresh_unconverged_alpha(oica_ctx* c, const int* act, int L_fin, int n_coarse, int vN) {
  cudaStream_t st = c->st;
  const int* cnt = c->Lact_dev.p;
  const bool tc = c->tc();
  c->Gfin.ensure((size_t)c->Ll * c->vNP);
  c->s4fin.ensure((size_t)c->Ll);
  c->cur_t = 0;
  // (the operand rows of the active runs already hold their final w: the last update wrote them)
  // no split-slot parts: they would depend on the global count, which other ranks may not join
  // here; the plain slot sums make alpha~ of a row the same for any GPU count
  run_step(c, act, L_fin, n_coarse, cnt, nullptr, false, false, false);
  const SlotPartials G = tc ? SlotPartials{c->Gp32.p, true} : SlotPartials{c->Gp.p, false};
  c->count(launch_slot_reduce(st, G, tc ? nullptr : c->s4p.p, c->S, c->Ll, c->vNP, L_fin, vN, c->Gfin.p, c->vNP,
                              c->s4fin.p, cnt));
  if (c->mshard()) {
    auto& nc = Nccl::get();
    c->exchange([&] { OICA_NCCL(nc.AllReduce(c->Gfin.p, c->Gfin.p, (size_t)L_fin * c->vNP, ncclFloat64, ncclSum, c->comm, st)); });
    if (!tc) c->exchange([&] { OICA_NCCL(nc.AllReduce(c->s4fin.p, c->s4fin.p, (size_t)L_fin, ncclFloat64, ncclSum, c->comm, st)); });
  }
  if (tc) c->count(launch_s4_from_g(st, c->eval_point(), act, c->Gfin.p, c->vNP, L_fin, vN, c->s4fin.p, cnt));
  c->count(launch_alpha_refresh(st, act, cnt, L_fin, c->s4fin.p, (double)c->Mg, c->alpha_old.p));
  check_launch();
}

// Active counts of every rank (hybrid mode): one all-gather of the device counter.
std::vector<int> gather_counts(oica_ctx* c) {
  const int W = c->world();
  c->tail.cnt_all.ensure((size_t)W);
  c->exchange([&] { OICA_NCCL(Nccl::get().AllGather(c->Lact_dev.p, c->tail.cnt_all.p, 1, ncclInt32, c->comm, c->st)); });
  std::vector<int> v((size_t)W);
  OICA_CUDA(cudaMemcpyAsync(v.data(), c->tail.cnt_all.p, sizeof(int) * W, cudaMemcpyDeviceToHost, c->st));
  c->wait();
  return v;
}

int hybrid_rows(const oica_ctx* c) {
  static const int env = [] { const char* e = getenv("OICA_HYBRID_ROWS"); return e ? atoi(e) : -1; }();
  return env >= 0 ? env : kHybridRowsPerRank * c->world();
}

// Hybrid tail: the T runs still active on all ranks (this rank's are
// act[0..L_local)) are all-gathered in rank order (C4) and iterated M-sharded: every rank runs
// all T rows over its share of the slots of its replicated X, one fp64 all-reduce of G per
// iteration, identical epilogue decisions everywhere; finished rows go back to
// their owners by global id.  Iterations t+1.. continue the component's count; returns this
// rank's share of the sum of active rows (rank 0 reports the tail).
int64_t run_hybrid_tail(oica_ctx* c, const int* act, int L_local, const std::vector<int>& counts, int& t, int K,
                        double tol, int kk, int vN, std::vector<std::pair<int, int>>& rows_at) {
  cudaStream_t st = c->st;
  auto& tb = c->tail;
  auto& nc = Nccl::get();
  const int W = c->world(), NP = c->vNP, R = vN + 4;
  const bool tc = c->tc();
  int T = 0, Pmax = 0;
  for (int v : counts) {
    T += v;
    Pmax = std::max(Pmax, v);
  }
  sync_x(c);
  tb.pack.ensure((size_t)Pmax * R);
  tb.pack_all.ensure((size_t)W * Pmax * R);
  tb.dense.ensure((size_t)T * R);
  tb.W64.ensure((size_t)T * vN);
  tb.alpha.ensure(T);
  tb.dprev.ensure(T);
  tb.ids.ensure(T);
  tb.iters.ensure(T);
  tb.act0.ensure(T);
  tb.act1.ensure(T);
  tb.state.ensure(T);
  tb.keep.ensure(T);
  tb.fine.ensure(T);
  tb.Gsum.ensure((size_t)T * NP);
  tb.s4sum.ensure(T);
  tb.hist.ensure(2 * ((size_t)K + 1));
  // C4: records of this rank's active rows, all-gathered; dense in rank order
  c->count(launch_tail_pack(st, act, c->Lact_dev.p, L_local, c->W64.p, c->alpha_old.p, tc ? c->dprev.p : nullptr,
                            c->fine_flags(), c->id_base, vN, tb.pack.p));
  c->exchange([&] { OICA_NCCL(nc.AllGather(tb.pack.p, tb.pack_all.p, (size_t)Pmax * R, ncclFloat64, c->comm, st)); });
  size_t off = 0;
  for (int r = 0; r < W; ++r) {
    if (counts[r] > 0)
      OICA_CUDA(cudaMemcpyAsync(tb.dense.p + off * R, tb.pack_all.p + (size_t)r * Pmax * R,
                                sizeof(double) * counts[r] * R, cudaMemcpyDeviceToDevice, st));
    off += counts[r];
  }
  c->count(launch_tail_unpack(st, tb.dense.p, T, vN, tb.W64.p, tb.alpha.p, tb.dprev.p, tb.fine.p, tb.state.p,
                              tb.keep.p, tb.ids.p));
  c->count(launch_compact(st, nullptr, tb.keep.p, tc ? tb.fine.p : nullptr, T, tb.act0.p, c->Lact_dev.p,
                          c->Lact_host));
  OICA_CUDA(cudaMemsetAsync(tb.hist.p, 0, sizeof(int) * 2 * ((size_t)K + 1), st));
  // tail slot plan: ~2 CTAs per SM on every rank for T rows; rank r owns slots [S r/W, S (r+1)/W)
  int tiles = (int)ceil_div(T, 128);
  if (tc && NP > 64) tiles = (int)round_up(tiles, 2);
  const int64_t S_want = std::min<int64_t>(kTailMaxSlots, (int64_t)W * std::max<int64_t>(1, ceil_div(2 * c->num_sms, tiles)));
  const int64_t slot_len = std::max<int64_t>(kSlotAlign, round_up(ceil_div(c->M, S_want), kSlotAlign));
  const int S_all = (int)ceil_div(c->M, slot_len);
  const int s0 = (int)((int64_t)S_all * c->cfg.rank / W), s1 = (int)((int64_t)S_all * (c->cfg.rank + 1) / W);
  const int s_cnt = s1 - s0;
  const int64_t m0 = (int64_t)s0 * slot_len, m1 = std::min<int64_t>(c->M, (int64_t)s1 * slot_len);
  const int64_t M_r = std::max<int64_t>(0, m1 - m0);
  if (tc) {
    tb.Gp32.ensure((size_t)std::max(S_all, 1) * T * NP);
    tb.Whi.ensure((size_t)T * NP);
    tb.Wlo.ensure((size_t)T * NP);
  } else {
    tb.Gp.ensure((size_t)std::max(s_cnt, 1) * T * NP);
    tb.s4p.ensure((size_t)std::max(s_cnt, 1) * T);
    tb.W32.ensure((size_t)T * NP);
  }
  EvalPoint ev = tc ? EvalPoint{tb.Whi.p, tb.Wlo.p, nullptr, NP} : EvalPoint{nullptr, nullptr, tb.W32.p, NP};
  Promotion pr = c->promotion();
  if (tc) {
    pr.fine = tb.fine.p;
    pr.dprev = tb.dprev.p;
  }
  // operand rows of the gathered runs (by tail index); the updates keep them current
  if (tc)
    c->count(launch_operand_f16x2(st, T, tb.W64.p, vN, NP, tb.fine.p, tb.Whi.p, tb.Wlo.p));
  else
    c->count(launch_operand_f32(st, T, tb.W64.p, vN, NP, tb.W32.p));
  c->wait();
  int L_ub = ((volatile int*)c->Lact_host)[0], nc_ub = ((volatile int*)c->Lact_host)[1];
  const int nc_first = nc_ub;
  int* a_cur = tb.act0.p;
  int* a_nxt = tb.act1.p;
  const int t_start = t;
  while (L_ub > 0 && t < K) {
    const int B = std::min(K - t, L_ub <= kBatchRows ? kBatch : 1);   // identical on every rank
    for (int b = 0; b < B; ++b) {
      ++t;
      const int* cnt = c->Lact_dev.p;
      cudaEvent_t e0 = c->event();
      c->cur_t = t;
      c->mark_pair();
      OICA_CUDA(cudaEventRecord(e0, st));
      int n = 0;
      if (s_cnt > 0 && tc)
        n = launch_step_tc(st, c->vXh, c->ldx, c->M, NP, tb.Whi.p, tb.Wlo.p, a_cur, nc_ub, L_ub, slot_len, S_all,
                           tb.Gp32.p, T, cnt, B > 1 && !c->split(), Upload{s0, s_cnt}, SplitOut{nullptr, 0, nullptr, 0},
                           c->xshift.p);
      else if (s_cnt > 0)
        n = launch_step_simt(st, c->vX + m0, c->vld, M_r, vN, NP, tb.W32.p, a_cur, L_ub, slot_len, s_cnt, kFlush,
                             tb.Gp.p, tb.s4p.p, T, cnt);
      check_launch();
      c->count(n);
      c->stats.step_launches += n;
      cudaEvent_t e1 = c->event();
      OICA_CUDA(cudaEventRecord(e1, st));
      SlotPartials part = tc ? SlotPartials{tb.Gp32.p + (size_t)s0 * T * NP, true} : SlotPartials{tb.Gp.p, false};
      c->count(launch_slot_reduce(st, part, tc ? nullptr : tb.s4p.p, s_cnt, T, NP, L_ub, vN, tb.Gsum.p, NP,
                                  tb.s4sum.p));
      c->exchange([&] { OICA_NCCL(nc.AllReduce(tb.Gsum.p, tb.Gsum.p, (size_t)L_ub * NP, ncclFloat64, ncclSum, c->comm, st)); });
      if (!tc) c->exchange([&] { OICA_NCCL(nc.AllReduce(tb.s4sum.p, tb.s4sum.p, (size_t)L_ub, ncclFloat64, ncclSum, c->comm, st)); });
      UpdateArgs u = update_args(c, SlotPartials{tb.Gsum.p, false}, tc ? nullptr : tb.s4sum.p, 1, T, a_cur, a_nxt,
                                 L_ub, tol, tb.hist.p);
      u.ev = ev;
      u.W64 = tb.W64.p;
      u.alpha_old = tb.alpha.p;
      u.iters = tb.iters.p;
      u.state = tb.state.p;
      u.keep = tb.keep.p;
      u.pr = pr;
      run_update(c, u);
      std::swap(a_cur, a_nxt);
      check_launch();
    }
    c->wait();
    L_ub = ((volatile int*)c->Lact_host)[0];
    nc_ub = ((volatile int*)c->Lact_host)[1];
  }
  if (L_ub > 0) {   // runs capped in the tail: alpha at their final w (A15; identical on every rank)
    const int* cnt = c->Lact_dev.p;
    if (s_cnt > 0 && tc)
      c->count(launch_step_tc(st, c->vXh, c->ldx, c->M, NP, tb.Whi.p, tb.Wlo.p, a_cur, nc_ub, L_ub, slot_len, S_all,
                              tb.Gp32.p, T, cnt, false, Upload{s0, s_cnt}, SplitOut{nullptr, 0, nullptr, 0}, c->xshift.p));
    else if (s_cnt > 0)
      c->count(launch_step_simt(st, c->vX + m0, c->vld, M_r, vN, NP, tb.W32.p, a_cur, L_ub, slot_len, s_cnt, kFlush,
                                tb.Gp.p, tb.s4p.p, T, cnt));
    SlotPartials part = tc ? SlotPartials{tb.Gp32.p + (size_t)s0 * T * NP, true} : SlotPartials{tb.Gp.p, false};
    c->count(launch_slot_reduce(st, part, tc ? nullptr : tb.s4p.p, s_cnt, T, NP, L_ub, vN, tb.Gsum.p, NP,
                                tb.s4sum.p));
    c->exchange([&] { OICA_NCCL(nc.AllReduce(tb.Gsum.p, tb.Gsum.p, (size_t)L_ub * NP, ncclFloat64, ncclSum, c->comm, st)); });
    if (!tc) c->exchange([&] { OICA_NCCL(nc.AllReduce(tb.s4sum.p, tb.s4sum.p, (size_t)L_ub, ncclFloat64, ncclSum, c->comm, st)); });
    if (tc) c->count(launch_s4_from_g(st, ev, a_cur, tb.Gsum.p, NP, L_ub, vN, tb.s4sum.p, cnt));
    c->count(launch_alpha_refresh(st, a_cur, cnt, L_ub, tb.s4sum.p, (double)c->Mg, tb.alpha.p));
    check_launch();
  }
  // finished (or capped) runs back to their owners
  c->count(launch_tail_scatter(st, T, tb.ids.p, tb.W64.p, tb.alpha.p, tb.iters.p, tb.state.p, c->id_base, c->Ll, vN,
                               c->W64.p, c->alpha_old.p, c->iters.p, c->state.p));
  check_launch();
  // work counters: rows entering tail iteration t' (T for the first)
  std::vector<int> hist(2 * ((size_t)K + 1), 0);
  OICA_CUDA(cudaMemcpyAsync(hist.data(), tb.hist.p, sizeof(int) * hist.size(), cudaMemcpyDeviceToHost, st));
  c->wait();
  int64_t sum_active = 0;
  for (int tt = t_start + 1; tt <= t; ++tt) {
    const int Lin = tt == t_start + 1 ? T : hist[2 * (tt - 1)];
    const int ncin = tt == t_start + 1 ? nc_first : hist[2 * (tt - 1) + 1];
    if (Lin <= 0) break;
    account_iteration(c, Lin, ncin, M_r);
    sum_active += Lin;
    rows_at[tt] = {Lin, ncin};
    ++c->stats.tail_iterations;
  }
  return c->cfg.rank == 0 ? sum_active : 0;
}

// The do-while of PAPER.md:241-256 for short iterations, on the device: a CUDA graph whose WHILE
// node runs [fused step over the active list act0 (grid sized for L_ub rows); fused update act0 ->
// act1 with copy-back, whose last block also sets the loop condition] until no run is active or
// t > K.  One graph launch (and one
// host wait) per component instead of a host round trip per batch of iterations; the kernels are
// those of the host-launched loop with the same upper-bound sizing, so results are bitwise equal
// (tests/test_gpu_parity.py::test_device_loop_bitwise).  Enqueues only (no host wait).
// Host wait for one event of the context's stream (single rank: no NCCL state to poll)
void wait_event(oica_ctx* c, cudaEvent_t ev) {
  (void)c;
  OICA_CUDA(cudaEventSynchronize(ev));
}

void ensure_loop_events(oica_ctx* c) {
  if (!c->loop_ev0[c->slot]) {
    OICA_CUDA(cudaEventCreate(&c->loop_ev0[c->slot]));
    OICA_CUDA(cudaEventCreate(&c->loop_ev1[c->slot]));
  }
}

// iterations per WHILE-body execution of the device-side loop
int loop_unroll() {
  static const int u = [] {
    const char* e = getenv("OICA_LOOP_UNROLL");
    const int v = e ? atoi(e) : kLoopUnroll;
    return v < 1 ? 1 : (v > 8 ? 8 : v);
  }();
  return u;
}

void enqueue_loop_graph(oica_ctx* c, int L_ub, int nc_ub, int K, double tol) {
  cudaStream_t st = c->st;
  c->loop_persistent = false;
  oica_ctx::LoopKey key;
  std::memset(&key, 0, sizeof key);   // (padding bytes take part in the comparison)
  key.X = c->vX;
  key.Xh = c->vXh;
  const void* bufs[12] = {c->act0.p, c->act1.p, c->W64.p, c->Whi.p, c->Wlo.p, c->W32.p, c->Gp32.p, c->Gsub.p,
                          c->Gp.p, c->s4p.p, c->hist.p, c->xshift.p};
  std::memcpy(key.buf, bufs, sizeof bufs);
  key.M = c->M;
  key.Mg = c->Mg;
  key.slot_len = c->slot_len;
  key.ldx = c->ldx;
  key.vld = c->vld;
  key.vN = c->vN;
  key.vNP = c->vNP;
  key.S = c->S;
  key.L_ub = L_ub;
  key.K = K;
  key.precision = c->precision;
  key.tol = tol;
  if (!(c->loop.valid && c->loop.key == key)) {
    c->loop.reset();
    // grid-size tiers: the loop over L_ub rows hands over to one sized for 2048, then 128, then 32
    // rows once that few remain (few-row iterations: tight grids, the few-row update path)
    std::vector<int> tiers{L_ub};
    for (int x : {2048, 128, 32})
      if (x < tiers.back()) tiers.push_back(x);
    const int nt = (int)tiers.size();
    OICA_CUDA(cudaGraphCreate(&c->loop.g, 0));
    std::vector<cudaGraphConditionalHandle> hs((size_t)nt);
    for (int i = 0; i < nt; ++i)   // the gate starts the first loop; each loop hands over to the next
      OICA_CUDA(cudaGraphConditionalHandleCreate(&hs[i], c->loop.g, 0, cudaGraphCondAssignDefault));
    cudaGraphNode_t prev = nullptr;
    add_loop_gate_node(c->loop.g, &prev, hs[0], c->Lact_dev.p, c->ctl.p, K);
    for (int i = 0; i < nt; ++i) {
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = hs[i];
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t wnode;
      OICA_CUDA(cudaGraphAddNode(&wnode, c->loop.g, prev ? &prev : nullptr, prev ? 1 : 0, &cp));
      prev = wnode;
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      OICA_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      try {
        const int* cnt = c->Lact_dev.p;
        int* gate = c->Lact_dev.p + 2;
        const int Lt = tiers[i];
        // the body holds kLoopUnroll iterations (a WHILE re-launch costs ~3 us, measured by
        // scripts/while_overhead.cu); copies after the first run only while the gate is open
        for (int j = 0; j < loop_unroll(); ++j) {
          const int* cs = j == 0 ? cnt : gate;
          run_step(c, c->act0.p, Lt, std::min(nc_ub, Lt), cs, cs, c->tc() && !c->split(), false);
          UpdateArgs u = update_args(c, c->partials(cnt, Lt), c->tc() ? nullptr : c->s4p.p, c->S, c->Ll, c->act0.p,
                                     c->act1.p, Lt, tol, c->hist.p);
          u.copy_back = 1;
          u.loop = hs[i];
          u.loop_next = i + 1 < nt ? hs[i + 1] : 0;
          u.loop_thr = i + 1 < nt ? tiers[i + 1] : 0;
          u.K_loop = K;
          u.gate_in = j == 0 ? nullptr : gate;
          u.gate_out = gate;
          run_update(c, u);
          check_launch();
        }
      } catch (...) {
        cudaGraph_t junk;
        cudaStreamEndCapture(st, &junk);
        c->loop.reset();
        throw;
      }
      cudaGraph_t captured;
      OICA_CUDA(cudaStreamEndCapture(st, &captured));
    }
    OICA_CUDA(cudaGraphInstantiate(&c->loop.x, c->loop.g, 0));
    c->loop.tiers = tiers;
    c->loop.unroll = loop_unroll();
    c->loop.key = key;
    c->loop.valid = true;
  }
  ensure_loop_events(c);
  OICA_CUDA(cudaEventRecord(c->loop_ev0[c->slot], st));
  OICA_CUDA(cudaGraphLaunch(c->loop.x, st));
  OICA_CUDA(cudaEventRecord(c->loop_ev1[c->slot], st));
}

// counters of a finished device-side loop of `iters` iterations (after the host wait); hh = the
// per-iteration history (rows entering iteration t at hh[2 (t - 1)]).  Launches counted as the
// graph ran them: the gate node, then per body execution of tier i `unroll` x (step + update
// [+ k_compact_iter above kUpdateCompactRows rows]), gated copies included
void finish_loop_graph(oica_ctx* c, int iters, int slot, const int* hh) {
  float ms = 0.f;
  OICA_CUDA(cudaEventElapsedTime(&ms, c->loop_ev0[slot], c->loop_ev1[slot]));
  c->stats.graph_ms += ms;
  if (c->loop_persistent) {
    c->count(1);
    c->stats.step_launches += 1;
    return;
  }
  const std::vector<int>& tiers = c->loop.tiers;
  const int nt = (int)tiers.size(), U = c->loop.unroll;
  std::vector<int> n_in((size_t)std::max(nt, 1), 0);   // iterations run by each tier's loop
  int ti = 0;
  for (int tt = 1; tt <= iters; ++tt) {
    ++n_in[(size_t)ti];
    const int out = tt < iters ? hh[2 * tt] : 0;   // rows left after iteration tt
    // hand-over: the next tier's loop runs at least one iteration before testing its threshold
    if (ti + 1 < nt && out <= tiers[(size_t)ti + 1]) ++ti;
  }
  int64_t launches = 1, steps = 0;
  for (int i = 0; i < nt; ++i) {
    const int64_t bodies = (n_in[(size_t)i] + U - 1) / U;
    const int per = 2 + (tiers[(size_t)i] > kUpdateCompactRows ? 1 : 0);
    launches += bodies * U * per;
    steps += bodies * U;
  }
  c->count((int)launches);
  c->stats.step_launches += steps;
}

// Tiny FP32 problems (the paper's own experiment sizes): the persistent cooperative loop
constexpr int64_t kPersistentMaxRows = 512;
bool persistent_loop_ok(const oica_ctx* c) {
  return !c->tc() && !c->reduced && c->Ll <= kPersistentMaxRows && c->M < kSimtShortM &&
         (c->vNP == 32 || c->vNP == 64);
}

void enqueue_loop_simt(oica_ctx* c, int K, double tol) {
  cudaStream_t st = c->st;
  ensure_loop_events(c);
  UpdateArgs u = update_args(c, SlotPartials{c->Gp.p, false}, c->s4p.p, c->S, c->Ll, c->act0.p, c->act1.p, (int)c->Ll,
                             tol, c->hist.p);
  u.copy_back = 1;
  OICA_CUDA(cudaEventRecord(c->loop_ev0[c->slot], st));
  launch_loop_simt(st, c->vX, c->vld, c->M, c->slot_len, c->S, kFlush, K, u, c->vNP, c->num_sms);
  check_launch();
  OICA_CUDA(cudaEventRecord(c->loop_ev1[c->slot], st));
  c->loop_persistent = true;
}

void extract_impl(oica_ctx* c, int32_t N_out, int32_t K, double tol, uint32_t flags, const double* W_prefix,
                  int32_t k_prefix, oica_result* out) {
  OICA_REQUIRE(c->X, OICA_ERR_STATE, "oica_set_data has not been called");
  OICA_REQUIRE(c->have_cand, OICA_ERR_STATE, "oica_init_candidates has not been called");
  OICA_REQUIRE(out, OICA_ERR_INVALID_ARGUMENT, "out is NULL");
  OICA_REQUIRE(K >= 1, OICA_ERR_INVALID_ARGUMENT, "max_iter must be >= 1");
  OICA_REQUIRE(tol > 0, OICA_ERR_INVALID_ARGUMENT, "tol must be > 0");
  OICA_REQUIRE(k_prefix >= 0 && k_prefix < N_out && N_out <= c->N, OICA_ERR_INVALID_ARGUMENT,
               "need 0 <= k_prefix < N_out <= N");
  OICA_REQUIRE(k_prefix == 0 || W_prefix, OICA_ERR_INVALID_ARGUMENT, "W_prefix is NULL");
  const int N = (int)c->N;
  cudaStream_t st = c->st;
  if (c->collective()) {   // collective call: every rank must pass the same arguments
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* p, size_t n) {
      const unsigned char* b = (const unsigned char*)p;
      for (size_t q = 0; q < n; ++q) h = (h ^ b[q]) * 1099511628211ull;   // FNV-1a
    };
    mix(&N_out, sizeof N_out);
    mix(&K, sizeof K);
    mix(&tol, sizeof tol);
    mix(&flags, sizeof flags);
    mix(&k_prefix, sizeof k_prefix);
    mix(&c->N, sizeof c->N);
    mix(&c->Mg, sizeof c->Mg);
    mix(&c->seed, sizeof c->seed);
    mix(&c->L, sizeof c->L);
    if (k_prefix > 0) mix(W_prefix, sizeof(double) * k_prefix * N);
    int64_t v[2] = {(int64_t)(h >> 2), -(int64_t)(h >> 2)}, r[2] = {0, 0};
    c->arghash.ensure(2);
    OICA_CUDA(cudaMemcpyAsync(c->arghash.p, v, sizeof v, cudaMemcpyHostToDevice, st));
    c->exchange([&] { OICA_NCCL(Nccl::get().AllReduce(c->arghash.p, c->arghash.p, 2, ncclInt64, ncclMax, c->comm, st)); });
    OICA_CUDA(cudaMemcpyAsync(r, c->arghash.p, sizeof r, cudaMemcpyDeviceToHost, st));
    c->wait();
    OICA_REQUIRE(r[0] == v[0] && r[1] == v[1], OICA_ERR_INVALID_ARGUMENT,
                 "ranks called oica_extract_components with different arguments");
  }
  if (k_prefix > 0)
    OICA_CUDA(cudaMemcpyAsync(c->Wacc.p, W_prefix, sizeof(double) * k_prefix * N, cudaMemcpyHostToDevice, st));
  out->n_extracted = k_prefix;
  out->stopped = 0;
  std::vector<double> w_host(N), b_host(N);
  ComponentRecord rec_h{};
  c->hist.ensure(2 * ((size_t)K + 1));
  const bool reduce = flags & OICA_REDUCE_X;
  if (reduce) {   // complement basis of the prefix (identity when there is none)
    if (k_prefix > 0) {
      complement_basis(W_prefix, k_prefix, N, c->Gh);
    } else {
      c->Gh.assign((size_t)N * N, 0.0);
      for (int n = 0; n < N; ++n) c->Gh[(size_t)n * N + n] = 1.0;
    }
    c->Wacc_scratch.ensure((size_t)N);
  }
  use_full_view(c);
  c->iter_log.clear();
  PhaseTrace trace;
  // Components are enqueued one ahead where nothing the host computes feeds the next one (the
  // device-side loop on one rank, no reduction, no Gaussianity stop): the GPU runs component k+1
  // while the host reads component k's record from its pinned slot, instead of idling between
  // components.  Elsewhere each component is finished before the next is enqueued.
  struct Comp {
    int k = 0, slot = 0;
    bool fast = false;
    int t = 0;
    std::vector<std::pair<int, int>> rows_at;
  };
  const bool ahead = !reduce && !(flags & OICA_STOP_ON_GAUSSIANITY) && !c->collective() && !(flags & OICA_EAGER) &&
                     (double)c->M * (double)c->vNP < kBatchMaxWork;
  trace.phases = !ahead;
  c->ensure_pin(K);
  for (int j = 0; j < 2; ++j)
    if (!c->comp_ev[j]) OICA_CUDA(cudaEventCreateWithFlags(&c->comp_ev[j], cudaEventDisableTiming));
  auto enqueue = [&](int k, Comp& cp) {
    const int i = k + 1;  // 1-based component index
    cp.k = k;
    trace.begin(i);
    const int j = cp.slot;
    c->slot = j;
    // Alg. 2 lines 4-12: iterate on X~ = G X in the d = N - k dimensional complement
    if (reduce && k > 0)
      use_reduced_view(c, N - k);
    else
      use_full_view(c);
    const int vN = c->vN;
    const int kk = c->reduced ? 0 : k;   // rows projected out per update (none in the reduced space)
    // a1: fresh candidates for this component (A8)
    if (c->reduced)
      c->count(launch_cand_basis(st, c->seed, i, c->id_base, c->Ll, N, c->Gdev.p, vN, c->W64.p, c->state.p,
                                 c->keep.p, c->fine.p, c->split() ? 1 : 0, c->dprev.p));
    else
      c->count(launch_cand_init(st, c->seed, i, c->id_base, c->Ll, N, c->Wacc.p, k, c->W64.p, c->state.p, c->keep.p,
                                c->fine.p, c->split() ? 1 : 0, c->dprev.p));
    // one rank, short iterations (the paper's own experiment sizes): the component -- draw,
    // device-side do-while, alpha refresh, selection, accept -- is enqueued without a host round
    // trip and its counters are read back once at the end (DESIGN.md §5 "iteration")
    const bool fast = !c->collective() && !c->reduced && !(flags & OICA_EAGER) &&
                      (double)c->M * (double)c->vNP < kBatchMaxWork;
    cp.fast = fast;
    c->count(launch_compact(st, nullptr, c->keep.p, c->fine_flags(), (int)c->Ll, c->act0.p, c->Lact_dev.p,
                            c->Lact_host, nullptr, c->hist.p));   // hist[0..1]: runs entering iteration 1
    OICA_CUDA(cudaMemsetAsync(c->nonfinite.p, 0, sizeof(int), st));
    c->count(launch_ctl_set(st, c->ctl.p, 1, kk));   // iteration t = 1, k accepted rows projected out
    build_operand(c, (int)c->Ll);
    if (!fast) c->wait();
    trace.mark("init");
    // fast: upper bounds (every kernel takes the true counts from the device)
    int L_act = fast ? (int)c->Ll : ((volatile int*)c->Lact_host)[0];
    int n_coarse = fast ? (c->split() ? 0 : (int)c->Ll) : ((volatile int*)c->Lact_host)[1];
    int* act = c->act0.p;
    int* act_next = c->act1.p;
    // a2-a6: the do-while of PAPER.md:241-256.  Iterations are enqueued in batches without a
    // host round trip once few rows remain (every kernel takes the true active count from the
    // device counters; the host value is an upper bound that sizes the grids); the per-iteration
    // counts are read back from `hist` afterwards.
    const int L0 = L_act, nc0 = n_coarse;
    int t = 0;
    int L_ub = L_act, nc_ub = n_coarse;
    // OICA_SHARD_HYBRID: the loop runs on the GLOBAL active count (ranks stay in step; a rank
    // without active rows idles) until it falls to hybrid_rows(), then the tail takes over
    // L-shard with a communicator (and hybrid) runs in lock step on the GLOBAL active count: the
    // split-slot parts of the step (common.cuh split_parts) depend on it, so every rank needs it
    // each iteration (one 4-byte all-reduce on the stream); a rank without active rows idles
    const bool hyb = c->hybrid();
    const bool lockstep = c->collective() && !c->mshard();
    std::vector<int> counts;
    int G_ub = L_ub;
    auto refresh = [&]() {   // all ranks' counts (host); true: hand the rest to the hybrid tail
      counts = gather_counts(c);
      G_ub = std::accumulate(counts.begin(), counts.end(), 0);
      return hyb && G_ub > 0 && G_ub <= hybrid_rows(c) && t < K;
    };
    if (lockstep) OICA_CUDA(cudaMemsetAsync(c->hist.p, 0, sizeof(int) * 2 * ((size_t)K + 1), st));
    bool to_tail = lockstep && refresh();
    if (fast) {   // the whole do-while on the device
      if (c->x_pending && c->tc()) {
        // a pipelined host upload is in flight (oica_set_data_host): iteration 1 is launched here,
        // its step piece by piece as the upload lands -- the kernels and sizes of
        // the graph body, so the same arithmetic -- and the graph continues from t = 2
        const int* cnt = c->Lact_dev.p;
        run_step(c, act, L_ub, nc_ub, cnt, cnt, c->tc() && !c->split(), false);
        UpdateArgs u = update_args(c, c->partials(cnt, L_ub), nullptr, c->S, c->Ll, act, c->act1.p, L_ub, tol,
                                   c->hist.p);
        u.copy_back = 1;
        run_update(c, u);
        check_launch();
      }
      sync_x(c);   // (the rest of the loop is a graph captured on the context stream)
      if (persistent_loop_ok(c) && !(flags & OICA_NO_PERSISTENT))
        enqueue_loop_simt(c, K, tol);      // tiny FP32 problems: one cooperative launch
      else
        enqueue_loop_graph(c, L_ub, nc_ub, K, tol);   // one graph launch
    }
    while (!fast && !to_tail && (lockstep ? G_ub : L_ub) > 0 && t < K) {
      // batches only where an iteration is short next to a host round trip (one row tile over
      // M samples: ~M NP 512 flop); elsewhere the exact count sizes every launch (grid, clusters)
      const bool short_iter = (double)c->M * (double)c->vNP < kBatchMaxWork;
      const int B = std::min(K - t, ((lockstep ? G_ub : L_ub) <= kBatchRows * (lockstep ? c->world() : 1) &&
                                     !c->mshard() && short_iter) ? kBatch : 1);
      trace.batch_begin();
      for (int b = 0; b < B; ++b) {
        ++t;
        const int* cnt = c->Lact_dev.p;
        const int* cnt_g = cnt;
        if (lockstep) {
          c->exchange([&] { OICA_NCCL(Nccl::get().AllReduce(c->Lact_dev.p, c->Lg.p, 1, ncclInt32, ncclSum, c->comm, st)); });
          cnt_g = c->Lg.p;
        }
        if (L_ub == 0) continue;   // lock step: this rank idles while others iterate
        c->cur_t = t;
        run_step(c, act, L_ub, nc_ub, cnt, cnt_g, B > 1 && c->tc() && !c->split(), true);
        const bool tc = c->tc();
        SlotPartials G = c->partials(cnt_g, L_ub);
        const double* s4 = tc ? nullptr : c->s4p.p;   // TC: alpha~ from the identity w_e . G (K3)
        int S = c->S;
        int64_t cap = c->Ll;
        if (c->mshard()) {  // one fp64 allreduce of (G, s4) per iteration; B == 1 here
          c->count(launch_slot_reduce(st, G, s4, c->S, c->Ll, c->vNP, L_ub, vN, c->Gsum.p, c->vNP, c->s4sum.p, cnt));
          auto& nc = Nccl::get();
          c->exchange([&] { OICA_NCCL(nc.AllReduce(c->Gsum.p, c->Gsum.p, (size_t)L_ub * c->vNP, ncclFloat64, ncclSum, c->comm, st)); });
          if (!tc) c->exchange([&] { OICA_NCCL(nc.AllReduce(c->s4sum.p, c->s4sum.p, (size_t)L_ub, ncclFloat64, ncclSum, c->comm, st)); });
          G = SlotPartials{c->Gsum.p, false};
          s4 = tc ? nullptr : c->s4sum.p;
          S = 1;
          cap = c->Ll;
        }
        // K3 + K4 in one launch: slot sums, eq. (5), projection, convergence, next operand rows,
        // compaction by the last block (DESIGN.md §5 "iteration")
        run_update(c, update_args(c, G, s4, S, cap, act, act_next, L_ub, tol, c->hist.p));
        std::swap(act, act_next);
        check_launch();
      }
      trace.batch_enqueued();
      c->wait();
      trace.batch_done();
      L_ub = ((volatile int*)c->Lact_host)[0];
      nc_ub = ((volatile int*)c->Lact_host)[1];
      if (lockstep) to_tail = refresh();
    }
    const int t_bulk = t;
    int64_t tail_active = 0;
    std::vector<std::pair<int, int>> rows_at((size_t)K + 2, {0, 0});   // (L_act, n_coarse) entering iteration t
    if (to_tail) tail_active = run_hybrid_tail(c, act, L_ub, counts, t, K, tol, kk, vN, rows_at);
    // Runs still active at the cap K carry alpha at their previous w (A15 holds only at a fixed
    // point); where they can be selected (reading A4: no run converged, or
    // OICA_INCLUDE_UNCONVERGED) rank them by alpha at their final w, as PAPER.md:257-258 does:
    // one more forward pass over those rows (L-shard / single GPU; M-shard sums ranks).
    // (fast: always enqueued -- its kernels do nothing when no run is active at the cap)
    if (fast || (!to_tail && L_ub > 0 && t >= K)) refresh_unconverged_alpha(c, act, L_ub, nc_ub, vN);
    trace.mark("iterate");
    int64_t sum_active = -1;   // fast: the selection takes it (and n_iter) from the device state
    if (!fast) {
      // per-iteration counts: entering iteration t' the active set had hist[t'-1] rows (t' >= 2)
      std::vector<int> hist(2 * (size_t)(t_bulk + 1), 0);
      if (t_bulk > 0) {
        OICA_CUDA(cudaMemcpyAsync(hist.data(), c->hist.p, sizeof(int) * 2 * (size_t)(t_bulk + 1),
                                  cudaMemcpyDeviceToHost, st));
        c->wait();
      }
      sum_active = 0;
      int t_exec = 0;
      for (int tt = 1; tt <= t_bulk; ++tt) {
        int Lin = tt == 1 ? L0 : hist[2 * (tt - 1)], ncin = tt == 1 ? nc0 : hist[2 * (tt - 1) + 1];
        if (Lin <= 0) break;
        account_iteration(c, Lin, ncin);
        sum_active += Lin;
        rows_at[tt] = {Lin, ncin};
        t_exec = tt;
      }
      if (to_tail) {   // the tail's rows were counted by rank 0 (the merge sums ranks)
        sum_active += tail_active;
        t_exec = t;
      }
      t = t_exec;
    }
    // a7: selection and accept
    sync_x(c);   // the exact-alpha pass reads X (a rank may reach here without running a step)
    const int* nconv_g = nullptr;
    if (c->collective() && !c->mshard()) {   // reading A4's "none converged" decided over all ranks
      c->count(launch_count_converged(st, c->state.p, (int)c->Ll, c->nconv.p));
      c->exchange([&] { OICA_NCCL(Nccl::get().AllReduce(c->nconv.p, c->nconv.p, 1, ncclInt32, ncclSum, c->comm, st)); });
      nconv_g = c->nconv.p;
    }
    c->count(launch_select_local(st, c->W64.p, c->alpha_old.p, c->state.p, c->iters.p, (int)c->Ll, c->id_base, vN,
                                 flags, c->vX, c->vld, c->M, c->cluster.p, c->pc.p, c->qc.p, c->csize.p, c->ups_max.p,
                                 c->counts.p, c->part.p, c->nblk_alpha, c->s4c.p, nconv_g));
    if (c->mshard())
      c->exchange([&] { OICA_NCCL(Nccl::get().AllReduce(c->s4c.p, c->s4c.p, kMaxClusters, ncclFloat64, ncclSum, c->comm, st)); });
    c->count(launch_select_finish(st, c->W64.p, c->iters.p, c->counts.p, c->pc.p, c->qc.p, c->csize.p, c->s4c.p,
                                  c->id_base, vN, (double)c->Mg, flags, sum_active, t, c->nonfinite.p, c->ctl.p,
                                  c->summary.p, c->wsum.p));
    const RankSummary* all = c->summary.p;
    const double* wall = c->wsum.p;
    int world = 1;
    if (c->collective() && !c->mshard()) {  // L-shard: one exchange per component (C1)
      auto& nc = Nccl::get();
      c->exchange([&] { OICA_NCCL(nc.AllGather(c->summary.p, c->summary_all.p, sizeof(RankSummary), ncclUint8, c->comm, st)); });
      c->exchange([&] { OICA_NCCL(nc.AllGather(c->wsum.p, c->wsum_all.p, (size_t)kMaxClusters * vN, ncclFloat64, c->comm, st)); });
      all = c->summary_all.p;
      wall = c->wsum_all.p;
      world = c->world();
    }
    // reduced: the merge works on b (vN-dim) with the Gaussianity threshold of the d-dimensional
    // problem, 2(d+1)d/M = 2(N-i+2)(N-i+1)/M (i_eff = 1); the accepted row is w = G^T b (line 28)
    c->count(launch_merge_accept(st, all, wall, world, vN, c->reduced ? 1 : i, (double)c->Mg, flags,
                                 c->reduced ? c->Wacc_scratch.p : c->Wacc.p, c->reduced ? 0 : k, c->rec.p,
                                 c->w_out.p));
    check_launch();
    OICA_CUDA(cudaMemcpyAsync(c->pin_rec(j), c->rec.p, sizeof(ComponentRecord), cudaMemcpyDeviceToHost, st));
    OICA_CUDA(cudaMemcpyAsync(c->pin_w(j), c->w_out.p, sizeof(double) * vN, cudaMemcpyDeviceToHost, st));
    if (fast) {
      OICA_CUDA(cudaMemcpyAsync(c->pin_ctl(j), c->ctl.p, sizeof(IterCtl), cudaMemcpyDeviceToHost, st));
      OICA_CUDA(cudaMemcpyAsync(c->pin_hist(j), c->hist.p, sizeof(int) * 2 * ((size_t)K + 1), cudaMemcpyDeviceToHost,
                                st));
    }
    OICA_CUDA(cudaEventRecord(c->comp_ev[j], st));   // this component's record is in the pinned slot
    cp.t = t;
    cp.rows_at = std::move(rows_at);
    if (ahead) trace.end();
  };
  // returns true where the Gaussianity test stops the extraction
  auto finish = [&](Comp& cp) -> bool {
    const int k = cp.k, i = k + 1, j = cp.slot;
    const bool fast = cp.fast;
    const int vN = c->vN;
    int t = cp.t;
    std::vector<std::pair<int, int>>& rows_at = cp.rows_at;
    if (ahead)
      wait_event(c, c->comp_ev[j]);   // (step / exchange events are read once, after the last component)
    else
      c->harvest_events();   // the component's one host wait on the fast path
    rec_h = *c->pin_rec(j);
    std::copy(c->pin_w(j), c->pin_w(j) + vN, b_host.begin());
    if (fast) {   // counters of the device-side loop
      t = c->pin_ctl(j)->t - 1;
      const int* hh = c->pin_hist(j);
      for (int tt = 1; tt <= t; ++tt) {
        const int Lin = hh[2 * (tt - 1)], ncin = hh[2 * (tt - 1) + 1];
        if (Lin <= 0) break;
        account_iteration(c, Lin, ncin, -1, false);
        rows_at[tt] = {Lin, ncin};
      }
      finish_loop_graph(c, t, j, hh);
    }
    // per-iteration log: every executed iteration; step_ms from its launch's events, or -1 for the
    // iterations of the device-side loop (not timed one by one)
    std::vector<double> step_ms_at((size_t)K + 2, -1.0);
    for (const auto& pr : c->pairs)
      if (pr.first >= 1 && pr.first <= K) step_ms_at[pr.first] = std::max(0.0, step_ms_at[pr.first]) + pr.second;
    for (int tt = 1; tt <= t; ++tt) {
      if (rows_at[tt].first <= 0) continue;
      const int Lin = rows_at[tt].first, ncin = rows_at[tt].second;
      oica_iteration_record r{};
      r.component = i;
      r.iteration = tt;
      r.L_act = Lin;
      r.fine_rows = Lin - ncin;
      r.step_ms = step_ms_at[tt];
      r.flops = (double)Lin * (4.0 * vN + 3.0) * (double)c->M;
      c->iter_log.push_back(r);
    }
    trace.mark("select");
    c->last_valid = true;
    if (rec_h.n_nonfinite > 0)
      throw Error(OICA_ERR_NONFINITE, "component " + std::to_string(i) + ": " + std::to_string(rec_h.n_nonfinite) +
                                          " candidate update(s) were not finite (non-finite data?)");
    if (rec_h.status != OICA_OK)
      throw Error((oica_status)rec_h.status,
                  rec_h.status == OICA_ERR_ALL_CANDIDATES_DEGENERATE ? "all candidates degenerate (A18)"
                                                                     : "no eligible candidate with alpha > -2 (A13)");
    if (c->reduced) {   // w = G^T b, canonical sign (A17), appended to W_acc
      for (int n = 0; n < N; ++n) {
        double acc = 0.0;
        for (int r = 0; r < vN; ++r) acc += c->Gh[(size_t)r * N + n] * b_host[r];
        w_host[n] = acc;
      }
      double nw = 0.0;
      for (int n = 0; n < N; ++n) nw += w_host[n] * w_host[n];
      nw = std::sqrt(nw);
      int jm = 0;
      for (int n = 1; n < N; ++n)
        if (std::fabs(w_host[n]) > std::fabs(w_host[jm])) jm = n;
      double sg = w_host[jm] < 0 ? -1.0 : 1.0;
      for (int n = 0; n < N; ++n) w_host[n] *= sg / nw;
      OICA_CUDA(cudaMemcpyAsync(c->Wacc.p + (size_t)k * N, w_host.data(), sizeof(double) * N, cudaMemcpyHostToDevice,
                                st));
      c->wait();
    } else {
      std::copy(b_host.begin(), b_host.begin() + N, w_host.begin());
    }
    c->last_vN = vN;
    if (c->reduced) c->Gh_last.assign(c->Gh.begin(), c->Gh.begin() + (size_t)vN * N);
    if (reduce) deflate_basis(c->Gh, N - k, N, c->reduced ? b_host.data() : w_host.data());
    bool stop = (flags & OICA_STOP_ON_GAUSSIANITY) && rec_h.gaussian;
    if (out->W && !stop) std::memcpy(out->W + (size_t)k * N, w_host.data(), sizeof(double) * N);
    if (out->alpha) out->alpha[k] = rec_h.w_alpha;
    if (out->objective) out->objective[k] = rec_h.w_objective;
    if (out->upsilon) out->upsilon[k] = rec_h.w_upsilon;
    if (out->index) out->index[k] = rec_h.q;
    if (out->iters) out->iters[k] = rec_h.iters;
    if (out->n_iter) out->n_iter[k] = rec_h.n_iter;
    if (out->cluster_size) out->cluster_size[k] = (int32_t)rec_h.cluster_size;
    if (out->n_converged) out->n_converged[k] = (int32_t)rec_h.n_conv;
    if (out->n_unconverged) out->n_unconverged[k] = (int32_t)rec_h.n_unconv;
    if (out->n_degenerate) out->n_degenerate[k] = (int32_t)rec_h.n_deg;
    if (out->sum_active) out->sum_active[k] = rec_h.sum_active;
    if (out->gaussian_flag) out->gaussian_flag[k] = (uint8_t)rec_h.gaussian;
    if (out->near_tie) out->near_tie[k] = (uint8_t)rec_h.near_tie;
    if (out->dim) out->dim[k] = vN;
    if (stop) {
      out->stopped = 1;
      return true;
    }
    out->n_extracted = k + 1;
    trace.mark("accept");
    trace.flush(i);
    return false;
  };
  if (ahead) {
    Comp cur, nxt;
    cur.slot = 0;
    enqueue(k_prefix, cur);
    for (int k = k_prefix; k < N_out; ++k) {
      if (k + 1 < N_out) {
        nxt = Comp{};
        nxt.slot = 1 - cur.slot;
        enqueue(k + 1, nxt);
      }
      if (finish(cur)) break;
      std::swap(cur, nxt);
    }
    c->harvest_events();
  } else {
    for (int k = k_prefix; k < N_out; ++k) {
      Comp cp;
      enqueue(k, cp);
      if (finish(cp)) break;
    }
  }
  use_full_view(c);
}

void set_data_impl(oica_ctx* c, const float* Xw, int64_t N, int64_t M_local, int64_t ld, int64_t M_global,
                   bool prepare = true) {
  OICA_REQUIRE(Xw, OICA_ERR_INVALID_ARGUMENT, "Xw is NULL");
  sync_x(c);   // a pending upload still writes the planes
  OICA_REQUIRE(N >= 1 && N <= 256, OICA_ERR_INVALID_ARGUMENT, "need 1 <= N <= 256");
  OICA_REQUIRE(M_local >= 1 && ld >= M_local, OICA_ERR_INVALID_ARGUMENT, "need M_local >= 1 and ld >= M_local");
  OICA_REQUIRE(M_global > N, OICA_ERR_INVALID_ARGUMENT, "need M_global > N");
  OICA_REQUIRE(c->mshard() ? M_global >= M_local : M_global == M_local, OICA_ERR_DIMENSION_MISMATCH,
               "M_global must equal M_local unless shard_mode = M");
  if (c->have_cand && N != c->N) c->have_cand = false;
  c->X = Xw;
  c->N = N;
  c->M = M_local;
  c->ld = ld;
  c->Mg = M_global;
  int req = c->cfg.precision;
  // AUTO: tensor cores once M is large enough that the fp16 rounding noise of the contraction
  // (~2^-12 / sqrt(M) relative in G) sits well below the 1e-10 convergence test.
  bool want_tc = req == OICA_PREC_TC || req == OICA_PREC_TC_SPLIT;
  bool tc = (want_tc || (req == OICA_PREC_AUTO && M_global >= kTcMinSamples)) && tc_supported((int)N);
  OICA_REQUIRE(!(want_tc && !tc), OICA_ERR_INVALID_ARGUMENT, "tensor-core step unsupported for this N");
  c->precision = tc ? (req == OICA_PREC_TC_SPLIT ? OICA_PREC_TC_SPLIT : OICA_PREC_TC) : OICA_PREC_FP32;
  c->NP = tc ? tc_np((int)N) : (N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
  plan_slots(c);
  c->stats.precision = c->precision;
  c->stats.slots = c->S;
  if (tc) {
    c->ldx = round_up(M_local, 128);
    c->Xh.ensure((size_t)c->NP * c->ldx);
    c->xshift.ensure((size_t)ceil_div(M_local, kShiftBlock));
    if (prepare) {
      c->count(launch_x_prepare_f16(c->st, Xw, ld, (int)N, M_local, (int)c->NP, c->ldx, c->Xh.p));
      c->count(launch_block_shift(c->st, Xw, ld, (int)N, M_local, 0, M_local, c->xshift.p));
      check_launch();
    }
  }
  use_full_view(c);
  if (c->have_cand) ensure_candidate_buffers(c);
}

}  // namespace

// ============================== C ABI ======================================================
extern "C" {

const char* oica_status_string(oica_status s) {
  switch (s) {
    case OICA_OK: return "OICA_OK";
    case OICA_ERR_INVALID_ARGUMENT: return "OICA_ERR_INVALID_ARGUMENT";
    case OICA_ERR_DIMENSION_MISMATCH: return "OICA_ERR_DIMENSION_MISMATCH";
    case OICA_ERR_RANK_DEFICIENT: return "OICA_ERR_RANK_DEFICIENT";
    case OICA_ERR_ALL_CANDIDATES_DEGENERATE: return "OICA_ERR_ALL_CANDIDATES_DEGENERATE";
    case OICA_ERR_DOMAIN: return "OICA_ERR_DOMAIN";
    case OICA_ERR_STATE: return "OICA_ERR_STATE";
    case OICA_ERR_UNSUPPORTED_DEVICE: return "OICA_ERR_UNSUPPORTED_DEVICE";
    case OICA_ERR_OUT_OF_MEMORY: return "OICA_ERR_OUT_OF_MEMORY";
    case OICA_ERR_CUDA: return "OICA_ERR_CUDA";
    case OICA_ERR_NCCL: return "OICA_ERR_NCCL";
    case OICA_ERR_NONFINITE: return "OICA_ERR_NONFINITE";
  }
  return "OICA_UNKNOWN_STATUS";
}

const char* oica_last_error(const oica_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

oica_status oica_nccl_unique_id(void* out) {
  if (!out) return OICA_ERR_INVALID_ARGUMENT;
  try {
    ncclUniqueId id;
    OICA_NCCL(Nccl::get().GetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return OICA_OK;
  } catch (const Error& e) {
    return e.status;
  }
}

oica_status oica_create(const oica_config* cfg, oica_ctx** out) {
  if (!cfg || !out) return OICA_ERR_INVALID_ARGUMENT;
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world || cfg->world > 64) return OICA_ERR_INVALID_ARGUMENT;
  if (cfg->world > 1 && !cfg->nccl_unique_id) return OICA_ERR_INVALID_ARGUMENT;
  if (cfg->shard_mode < OICA_SHARD_L || cfg->shard_mode > OICA_SHARD_HYBRID) return OICA_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  oica_ctx* c = new (std::nothrow) oica_ctx();
  if (!c) return OICA_ERR_OUT_OF_MEMORY;
  c->cfg = *cfg;
  oica_status s = guard(c, [&] {
    cudaDeviceProp prop;
    OICA_CUDA(cudaGetDeviceProperties(&prop, cfg->device));
    OICA_REQUIRE(prop.major == 10 && prop.minor == 0, OICA_ERR_UNSUPPORTED_DEVICE,
                 std::string("liboica is built for sm_100a (B200); device is ") + prop.name);
    c->num_sms = prop.multiProcessorCount;
    if (cfg->stream) {
      c->st = (cudaStream_t)cfg->stream;
    } else {
      OICA_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    OICA_CUDA(cudaHostAlloc((void**)&c->Lact_host, 2 * sizeof(int), cudaHostAllocMapped));
    if (const char* e = getenv("OICA_NCCL_TIMEOUT_S")) c->nccl_timeout_s = std::max(1.0, atof(e));
    if (cfg->world > 1 || cfg->nccl_unique_id) {
      ncclUniqueId id;
      std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
      OICA_NCCL(Nccl::get().CommInitRank(&c->comm, cfg->world, id, cfg->rank));
    }
  });
  if (s != OICA_OK) {
    oica_destroy(c);
    return s;
  }
  *out = c;
  return OICA_OK;
}

oica_status oica_destroy(oica_ctx* c) {
  if (!c) return OICA_OK;
  cudaSetDevice(c->cfg.device);
  if (c->st) cudaStreamSynchronize(c->st);
  if (c->comm) Nccl::get().CommDestroy(c->comm);
  for (auto e : c->ev) cudaEventDestroy(e);
  for (auto& e : c->xev) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c->loop.reset();
  for (int j = 0; j < 2; ++j) {
    if (c->loop_ev0[j]) cudaEventDestroy(c->loop_ev0[j]);
    if (c->loop_ev1[j]) cudaEventDestroy(c->loop_ev1[j]);
    if (c->comp_ev[j]) cudaEventDestroy(c->comp_ev[j]);
  }
  if (c->pin) cudaFreeHost(c->pin);
  if (c->Lact_host) cudaFreeHost(c->Lact_host);
  if (c->cst) {
    cudaStreamSynchronize(c->cst);
    cudaStreamDestroy(c->cst);
  }
  if (c->x_ready_ev) cudaEventDestroy(c->x_ready_ev);
  for (auto e : c->piece_ev) cudaEventDestroy(e);
  if (c->st_ev) cudaEventDestroy(c->st_ev);
#ifdef OICA_EXPERIMENTS
  if (c->st2) {
    cudaStreamSynchronize(c->st2);
    cudaStreamDestroy(c->st2);
  }
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->green.ok) {
    GreenApi& api = GreenApi::get();
    cudaEventDestroy(c->green.fork);
    cudaEventDestroy(c->green.jA);
    cudaEventDestroy(c->green.jB);
    api.StreamDestroy(c->green.sA);
    api.StreamDestroy(c->green.sB);
    api.GreenCtxDestroy(c->green.gA);
    api.GreenCtxDestroy(c->green.gB);
  }
#endif
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  delete c;
  return OICA_OK;
}

oica_status oica_whiten(oica_ctx* c, const float* X, int64_t N, int64_t M, int64_t ld, double eig_floor, float* Xw,
                        int64_t ld_out, double* mean_out, double* V_out, double* eig_out) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] {
    OICA_REQUIRE(X && Xw, OICA_ERR_INVALID_ARGUMENT, "X / Xw is NULL");
    OICA_REQUIRE(N >= 1 && N <= 256 && M > N && ld >= M && ld_out >= M, OICA_ERR_INVALID_ARGUMENT,
                 "need 1 <= N <= 256, M > N, ld >= M, ld_out >= M");
    OICA_REQUIRE(eig_floor >= 0, OICA_ERR_INVALID_ARGUMENT, "eig_floor < 0");
    int n = (int)N;
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(64, M / 8192));
    c->wh_mean.ensure(n);
    c->wh_part.ensure((size_t)nsplit * n * n);
    c->wh_C.ensure((size_t)n * n);
    c->wh_V.ensure((size_t)n * n);
    c->count(launch_row_mean(c->st, X, ld, n, M, c->wh_mean.p));
    c->count(launch_covariance(c->st, X, ld, n, M, c->wh_mean.p, c->wh_part.p, nsplit, c->wh_C.p));
    check_launch();
    std::vector<double> C((size_t)n * n), mean(n);
    OICA_CUDA(cudaMemcpyAsync(C.data(), c->wh_C.p, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->st));
    OICA_CUDA(cudaMemcpyAsync(mean.data(), c->wh_mean.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->st));
    OICA_CUDA(cudaStreamSynchronize(c->st));
    for (int i = 0; i < n; ++i)  // symmetrise
      for (int j = i + 1; j < n; ++j) C[(size_t)i * n + j] = C[(size_t)j * n + i] = 0.5 * (C[(size_t)i * n + j] + C[(size_t)j * n + i]);
    std::vector<double> d, E;
    jacobi_eigh(C, n, d, E);
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return d[a] > d[b]; });
    double dmax = d[order[0]], dmin = d[order[n - 1]];
    OICA_REQUIRE(dmin > 0 && dmin >= eig_floor * dmax, OICA_ERR_RANK_DEFICIENT,
                 "covariance eigenvalue below eig_floor * max (A11)");
    std::vector<double> V((size_t)n * n), ev(n);
    for (int r = 0; r < n; ++r) {
      int k = order[r];
      int jm = 0;
      double am = -1;
      for (int j = 0; j < n; ++j)
        if (std::fabs(E[(size_t)j * n + k]) > am) { am = std::fabs(E[(size_t)j * n + k]); jm = j; }
      double sg = E[(size_t)jm * n + k] < 0 ? -1.0 : 1.0;   // largest-|entry| positive
      double sc = sg / std::sqrt(d[k]);
      for (int j = 0; j < n; ++j) V[(size_t)r * n + j] = sc * E[(size_t)j * n + k];   // V = D^-1/2 E^T
      ev[r] = d[k];
    }
    OICA_CUDA(cudaMemcpyAsync(c->wh_V.p, V.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, c->st));
    c->count(launch_apply_whitening(c->st, X, ld, n, M, c->wh_mean.p, c->wh_V.p, Xw, ld_out));
    check_launch();
    c->wait();
    if (mean_out) std::memcpy(mean_out, mean.data(), sizeof(double) * n);
    if (V_out) std::memcpy(V_out, V.data(), sizeof(double) * n * n);
    if (eig_out) std::memcpy(eig_out, ev.data(), sizeof(double) * n);
  });
}

oica_status oica_set_data(oica_ctx* c, const float* Xw, int64_t N, int64_t M_local, int64_t ld, int64_t M_global) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] { set_data_impl(c, Xw, N, M_local, ld, M_global); });
}

oica_status oica_set_data_host(oica_ctx* c, const float* Xh, int64_t N, int64_t M_local, int64_t ld, int64_t M_global) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] {
    OICA_REQUIRE(Xh && N >= 1 && M_local >= 1 && ld >= M_local, OICA_ERR_INVALID_ARGUMENT, "bad host data");
    c->Xown.ensure((size_t)N * M_local);
    set_data_impl(c, c->Xown.p, N, M_local, M_local, M_global, /*prepare=*/false);
    if (!c->cst) {
      OICA_CUDA(cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking));
      OICA_CUDA(cudaEventCreateWithFlags(&c->x_ready_ev, cudaEventDisableTiming));
      OICA_CUDA(cudaEventCreateWithFlags(&c->st_ev, cudaEventDisableTiming));
    }
    // the upload may overwrite X and its plane only after all work already queued on the
    // context stream (which may still read them)
    OICA_CUDA(cudaEventRecord(c->st_ev, c->st));
    OICA_CUDA(cudaStreamWaitEvent(c->cst, c->st_ev, 0));
    // pieces of whole slots (~16 per upload) so the first step can start on the first piece
    const int64_t M = M_local;
    // (and >= ~2 waves of CTAs per piece launch at the first iteration's row count)
    int64_t spp = std::max<int64_t>(1, c->S / 16);
    if (c->have_cand) spp = std::max<int64_t>(spp, ceil_div(2 * c->num_sms, ceil_div(c->Ll, 128)));
    c->piece_len = c->tc() ? c->slot_len * std::min<int64_t>(spp, c->S) : M;
    c->pieces = (int)ceil_div(M, c->piece_len);
    while ((int)c->piece_ev.size() < c->pieces) {
      cudaEvent_t e;
      OICA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->piece_ev.push_back(e);
    }
    for (int p = 0; p < c->pieces; ++p) {
      const int64_t m0 = p * c->piece_len, m1 = std::min(M, m0 + c->piece_len);
      OICA_CUDA(cudaMemcpy2DAsync(c->Xown.p + m0, sizeof(float) * M, Xh + m0, sizeof(float) * ld, sizeof(float) * (m1 - m0),
                                  (size_t)N, cudaMemcpyHostToDevice, c->cst));
      if (c->tc()) {
        c->count(launch_x_prepare_f16(c->cst, c->Xown.p, M, (int)N, M, (int)c->NP, c->ldx, c->Xh.p, m0,
                                      p == c->pieces - 1 ? c->ldx : m1));
        c->count(launch_block_shift(c->cst, c->Xown.p, M, (int)N, M, m0, m1, c->xshift.p));   // m0: whole slots
      }
      OICA_CUDA(cudaEventRecord(c->piece_ev[p], c->cst));
    }
    check_launch();
    OICA_CUDA(cudaEventRecord(c->x_ready_ev, c->cst));
    c->x_pending = true;
  });
}

oica_status oica_distribute_data(oica_ctx* c, const float* X_root, int64_t N, int64_t M_global, int64_t ld_root,
                                 float* X_out, int64_t ld_out, int32_t root) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] {
    const int W = c->cfg.world, r = c->cfg.rank;
    OICA_REQUIRE(N >= 1 && N <= 256 && M_global > N && X_out && root >= 0 && root < W, OICA_ERR_INVALID_ARGUMENT,
                 "need 1 <= N <= 256, M_global > N, X_out, 0 <= root < world");
    OICA_REQUIRE(r != root || (X_root && ld_root >= M_global), OICA_ERR_INVALID_ARGUMENT,
                 "root: X_root NULL or ld_root < M_global");
    const bool msh = c->cfg.shard_mode == OICA_SHARD_M && W > 1;
    const int64_t lo = msh ? M_global * r / W : 0, hi = msh ? M_global * (r + 1) / W : M_global;
    OICA_REQUIRE(ld_out >= hi - lo, OICA_ERR_INVALID_ARGUMENT, "ld_out < this rank's sample count");
    cudaStream_t st = c->st;
    if (!c->comm) {   // one rank: a plain device copy (nothing to distribute)
      if (X_out != X_root)
        OICA_CUDA(cudaMemcpy2DAsync(X_out, sizeof(float) * ld_out, X_root, sizeof(float) * ld_root,
                                    sizeof(float) * M_global, (size_t)N, cudaMemcpyDeviceToDevice, st));
      c->wait();
      return;
    }
    auto& nc = Nccl::get();
    if (!msh) {   // replicated X (L-shard / hybrid): broadcast from root
      if (ld_root == M_global && ld_out == M_global) {
        c->exchange([&] {
          OICA_NCCL(nc.Broadcast(r == root ? X_root : X_out, X_out, (size_t)N * M_global, ncclFloat32, root, c->comm, st));
        });
      } else {   // strided rows: one broadcast per row, grouped
        c->exchange([&] {
          OICA_NCCL(nc.GroupStart());
          for (int64_t n = 0; n < N; ++n)
            OICA_NCCL(nc.Broadcast(r == root ? X_root + n * ld_root : X_out + n * ld_out, X_out + n * ld_out,
                                   (size_t)M_global, ncclFloat32, root, c->comm, st));
          OICA_NCCL(nc.GroupEnd());
        });
      }
    } else {   // M-shard: rank q receives the samples [q M/W, (q+1) M/W) of every row from root
      c->exchange([&] {
        OICA_NCCL(nc.GroupStart());
        if (r == root) {
          for (int q = 0; q < W; ++q) {
            const int64_t ql = M_global * q / W, qh = M_global * (q + 1) / W;
            if (q == root || qh <= ql) continue;
            for (int64_t n = 0; n < N; ++n)
              OICA_NCCL(nc.Send(X_root + n * ld_root + ql, (size_t)(qh - ql), ncclFloat32, q, c->comm, st));
          }
        } else if (hi > lo) {
          for (int64_t n = 0; n < N; ++n)
            OICA_NCCL(nc.Recv(X_out + n * ld_out, (size_t)(hi - lo), ncclFloat32, root, c->comm, st));
        }
        OICA_NCCL(nc.GroupEnd());
      });
      if (r == root && hi > lo)
        OICA_CUDA(cudaMemcpy2DAsync(X_out, sizeof(float) * ld_out, X_root + lo, sizeof(float) * ld_root,
                                    sizeof(float) * (hi - lo), (size_t)N, cudaMemcpyDeviceToDevice, st));
    }
    c->wait();
    c->harvest_events();
  });
}

oica_status oica_init_candidates(oica_ctx* c, uint64_t seed, int64_t L) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] {
    OICA_REQUIRE(c->X, OICA_ERR_STATE, "oica_set_data has not been called");
    OICA_REQUIRE(L >= 1 && L < (1 << 24), OICA_ERR_INVALID_ARGUMENT, "need 1 <= L < 2^24");
    int w = c->mshard() ? 1 : c->cfg.world, r = c->mshard() ? 0 : c->cfg.rank;
    c->seed = seed;
    c->L = L;
    c->id_base = L * r / w;
    c->Ll = L * (r + 1) / w - c->id_base;
    OICA_REQUIRE(c->Ll >= 1, OICA_ERR_INVALID_ARGUMENT, "fewer candidates than ranks");
    ensure_candidate_buffers(c);
    c->have_cand = true;
    c->last_valid = false;
  });
}

oica_status oica_extract_components(oica_ctx* c, int32_t N_out, int32_t K, double tol, uint32_t flags,
                                    const double* W_prefix, int32_t k_prefix, oica_result* out) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] { extract_impl(c, N_out, K, tol, flags, W_prefix, k_prefix, out); });
}

oica_status oica_fixed_point_step(oica_ctx* c, const double* W_dev, int64_t L, double* G_dev, double* s4_dev) {
  return oica_fixed_point_step_mixed(c, W_dev, L, nullptr, G_dev, s4_dev);
}

oica_status oica_fixed_point_step_mixed(oica_ctx* c, const double* W_dev, int64_t L, const uint8_t* fine_host,
                                        double* G_dev, double* s4_dev) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] {
    OICA_REQUIRE(c->X && c->have_cand, OICA_ERR_STATE, "set_data and init_candidates first");
    OICA_REQUIRE(W_dev && G_dev && s4_dev && L >= 1 && L <= c->Ll, OICA_ERR_INVALID_ARGUMENT, "bad arguments");
    // per-row precision: coarse rows first (the compaction's order), n_coarse of them
    int n_coarse = c->split() ? 0 : (int)L;
    std::vector<uint8_t> fl;
    if (fine_host && c->tc()) {
      fl.assign(fine_host, fine_host + L);
      for (auto& f : fl) f = f ? 1 : 0;
      n_coarse = (int)(std::find(fl.begin(), fl.end(), (uint8_t)1) - fl.begin());
      OICA_REQUIRE(std::find(fl.begin() + n_coarse, fl.end(), (uint8_t)0) == fl.end(), OICA_ERR_INVALID_ARGUMENT,
                   "fine rows must follow every coarse row");
    }
    // stage caller rows through the fp64 master (identity active list)
    OICA_CUDA(cudaMemcpyAsync(c->W64.p, W_dev, sizeof(double) * L * c->N, cudaMemcpyDeviceToDevice, c->st));
    OICA_CUDA(cudaMemsetAsync(c->keep.p, 1, L, c->st));
    if (!fl.empty())
      OICA_CUDA(cudaMemcpyAsync(c->fine.p, fl.data(), L, cudaMemcpyHostToDevice, c->st));
    else
      OICA_CUDA(cudaMemsetAsync(c->fine.p, c->split() ? 1 : 0, L, c->st));   // one precision for all rows
    c->count(launch_compact(c->st, nullptr, c->keep.p, nullptr, (int)L, c->act0.p, c->Lact_dev.p, nullptr));
    build_operand(c, (int)L);
    run_step(c, c->act0.p, (int)L, n_coarse, nullptr, nullptr, false, true);
    account_iteration(c, (int)L, n_coarse);
    bool tc = c->tc();
    c->count(launch_slot_reduce(c->st, c->partials(nullptr, (int)L), tc ? nullptr : c->s4p.p, c->S, c->Ll, (int)c->NP, (int)L,
                                (int)c->N, G_dev, (int)c->N, s4_dev));
    if (tc) c->count(launch_s4_from_g(c->st, c->eval_point(), nullptr, G_dev, (int)c->N, (int)L, (int)c->N, s4_dev));
    check_launch();
    c->harvest_events();
  });
}

oica_status oica_draw_candidates(oica_ctx* c, int32_t i, const double* W_acc, int32_t k, double* W_dev) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] {
    OICA_REQUIRE(c->have_cand, OICA_ERR_STATE, "init_candidates first");
    OICA_REQUIRE(i >= 1 && k >= 0 && k < c->N && (k == 0 || W_acc) && W_dev, OICA_ERR_INVALID_ARGUMENT,
                 "bad arguments");
    if (k > 0)
      OICA_CUDA(cudaMemcpyAsync(c->Wacc.p, W_acc, sizeof(double) * k * c->N, cudaMemcpyHostToDevice, c->st));
    c->count(launch_cand_init(c->st, c->seed, i, c->id_base, c->Ll, (int)c->N, c->Wacc.p, k, W_dev, c->state.p,
                              c->keep.p, nullptr, 0, nullptr));
    check_launch();
    OICA_CUDA(cudaStreamSynchronize(c->st));
    c->last_valid = false;
  });
}

oica_status oica_get_candidates(oica_ctx* c, double* W, double* alpha, int32_t* iters, uint8_t* state, int64_t* L_local,
                                int64_t* id_base) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] {
    OICA_REQUIRE(c->have_cand, OICA_ERR_STATE, "init_candidates first");
    if (L_local) *L_local = c->Ll;
    if (id_base) *id_base = c->id_base;
    if (!(W || alpha || iters || state)) return;
    OICA_REQUIRE(c->last_valid, OICA_ERR_STATE, "no extracted component yet");
    std::vector<double> Wb;
    const bool red = c->last_vN != (int)c->N;   // rows are b in the reduced basis: return w = G^T b
    if (W && !red) OICA_CUDA(cudaMemcpyAsync(W, c->W64.p, sizeof(double) * c->Ll * c->N, cudaMemcpyDeviceToHost, c->st));
    if (W && red) {
      Wb.resize((size_t)c->Ll * c->last_vN);
      OICA_CUDA(cudaMemcpyAsync(Wb.data(), c->W64.p, sizeof(double) * Wb.size(), cudaMemcpyDeviceToHost, c->st));
    }
    if (alpha) OICA_CUDA(cudaMemcpyAsync(alpha, c->alpha_old.p, sizeof(double) * c->Ll, cudaMemcpyDeviceToHost, c->st));
    if (iters) OICA_CUDA(cudaMemcpyAsync(iters, c->iters.p, sizeof(int32_t) * c->Ll, cudaMemcpyDeviceToHost, c->st));
    if (state) OICA_CUDA(cudaMemcpyAsync(state, c->state.p, c->Ll, cudaMemcpyDeviceToHost, c->st));
    OICA_CUDA(cudaStreamSynchronize(c->st));
    if (W && red) {
      const int N = (int)c->N, d = c->last_vN;
      for (int64_t l = 0; l < c->Ll; ++l)
        for (int n = 0; n < N; ++n) {
          double acc = 0.0;
          for (int r = 0; r < d; ++r) acc += Wb[(size_t)l * d + r] * c->Gh_last[(size_t)r * N + n];
          W[(size_t)l * N + n] = acc;
        }
    }
  });
}

oica_status oica_get_iteration_log(oica_ctx* c, oica_iteration_record* out, int64_t cap, int64_t* n) {
  if (!c || !n || (cap > 0 && !out)) return OICA_ERR_INVALID_ARGUMENT;
  *n = (int64_t)c->iter_log.size();
  for (int64_t k = 0; k < std::min<int64_t>(cap, *n); ++k) out[k] = c->iter_log[(size_t)k];
  return OICA_OK;
}

oica_status oica_get_stats(oica_ctx* c, oica_stats* out) {
  if (!c || !out) return OICA_ERR_INVALID_ARGUMENT;
  *out = c->stats;
  return OICA_OK;
}

oica_status oica_reset_stats(oica_ctx* c) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  int p = c->stats.precision, s = c->stats.slots;
  c->stats = oica_stats{};
  c->stats.precision = p;
  c->stats.slots = s;
  return OICA_OK;
}

oica_status oica_synchronize(oica_ctx* c) {
  if (!c) return OICA_ERR_INVALID_ARGUMENT;
  return guard(c, [&] { c->wait(); });
}

oica_status oica_slot_plan(int32_t precision, int64_t M_global, int64_t M_local, int64_t* slot_len,
                           int32_t* S_local) {
  if (!slot_len || !S_local || M_global < 1 || M_local < 1 || M_local > M_global || precision < OICA_PREC_AUTO ||
      precision > OICA_PREC_TC_SPLIT)
    return OICA_ERR_INVALID_ARGUMENT;
  int s = 0;
  const bool fp32 = precision == OICA_PREC_FP32 || (precision == OICA_PREC_AUTO && M_global < kTcMinSamples);
  plan_slots_for(M_global, M_local, fp32, slot_len, &s);
  *S_local = s;
  return OICA_OK;
}

oica_status oica_split_parts(int32_t L_global, int32_t S, int32_t* P) {
  if (!P || L_global < 0 || S < 1) return OICA_ERR_INVALID_ARGUMENT;
  *P = split_parts(L_global, S);
  return OICA_OK;
}

oica_status oica_complement_basis(const double* W, int32_t k, int32_t N, double* G) {
  if (!G || N < 1 || N > 4096 || k < 0 || k >= N || (k > 0 && !W)) return OICA_ERR_INVALID_ARGUMENT;
  std::vector<double> g;
  complement_basis(W, k, N, g);
  std::memcpy(G, g.data(), sizeof(double) * g.size());
  return OICA_OK;
}

oica_status oica_deflate_basis(double* G, int32_t d, int32_t N, const double* b, double* G_out) {
  if (!G || !b || !G_out || d < 2 || N < d) return OICA_ERR_INVALID_ARGUMENT;
  std::vector<double> g(G, G + (size_t)d * N);
  deflate_basis(g, d, N, b);
  std::memcpy(G_out, g.data(), sizeof(double) * g.size());
  return OICA_OK;
}

oica_status oica_merge_records(const oica_cluster_record* records, const double* w, int32_t n, int32_t N,
                               int32_t* winner, int64_t* merged_size, uint8_t* near_tie) {
  if (!records || !w || n < 0 || N < 1 || !winner) return OICA_ERR_INVALID_ARGUMENT;
  std::vector<int32_t> group((size_t)std::max(n, 1));
  MergeOut m = merge_records(records, w, n, N, group.data(), false, kClusterDelta, kNearTieRel);
  *winner = m.winner;
  if (merged_size) *merged_size = m.merged_size;
  if (near_tie) *near_tie = m.near_tie;
  return m.winner >= 0 ? OICA_OK : OICA_ERR_DOMAIN;
}

}  // extern "C"
