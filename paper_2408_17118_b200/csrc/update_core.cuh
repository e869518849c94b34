// Device code of the fp64 update (K3) and compaction (K4) shared by the update kernels
// (k_candidates.cu) and the persistent small-problem loop (k_loop_simt.cu): ONE definition of the
// arithmetic, so a row's result is bitwise the same whichever kernel runs it.  Internal.
#pragma once
#include <cuda_fp16.h>

#include "kernels.cuh"

namespace oica {
namespace upd {

constexpr int kMaxV = 8;  // 256 / 32 coordinates per lane

// c[b] <- warp_sum(c[b]) for every b, the butterfly stages issued value-interleaved (up to 8 values
// per stage): each value sees warp_sum's own sequence of adds (bitwise the same sums), but the
// shuffles of different values overlap -- one value after the other is a chain of 5 shuffle + add
// latencies per value (the compiler does not interleave them: measured)
template <int RB>
__device__ __forceinline__ void warp_sum_many(double (&c)[RB]) {
  constexpr int G = RB < 8 ? RB : 8;
#pragma unroll
  for (int b0 = 0; b0 < RB; b0 += G) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double t[G];
#pragma unroll
      for (int b = 0; b < G; ++b) t[b] = __shfl_xor_sync(0xffffffffu, c[b0 + b], o);
#pragma unroll
      for (int b = 0; b < G; ++b) c[b0 + b] += t[b];
    }
  }
}

// v <- v - E v with E = Wacc^T Wacc: all coefficients w_k . v are
// taken from the incoming v (one projection, as written in the paper).
template <int V>
__device__ __forceinline__ void project_warp(double (&v)[V], const double* __restrict__ Wacc, int k,
                                             int N, int lane) {
  double h[V];
#pragma unroll
  for (int u = 0; u < V; ++u) h[u] = 0.0;
  // rows in blocks of RB: their loads and warp reductions are independent (latency-bound
  // otherwise when few rows run); same operations in the same order per row (h accumulates the
  // rows in row order for any RB).  RB x V bounded (registers: 8 coordinates per lane fill them)
  constexpr int RB = V >= 8 ? 1 : 8 / V;
  for (int r0 = 0; r0 < k; r0 += RB) {
    const int nb = min(RB, k - r0);
    double c[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      c[b] = 0.0;
      if (b < nb) {
        const double* wr = Wacc + (int64_t)(r0 + b) * N;
#pragma unroll
        for (int u = 0; u < V; ++u) {
          int n = lane + 32 * u;
          if (n < N) c[b] += __ldg(wr + n) * v[u];
        }
      }
    }
    warp_sum_many<RB>(c);
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      if (b < nb) {
        const double* wr = Wacc + (int64_t)(r0 + b) * N;
#pragma unroll
        for (int u = 0; u < V; ++u) {
          int n = lane + 32 * u;
          if (n < N) h[u] += c[b] * __ldg(wr + n);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < V; ++u) v[u] -= h[u];
}

// sum_{j < n} v(j) in order j = 0, 1, ... (fp64), loads issued 8 at a time: with few active
// rows the epilogue is a chain of dependent adds over S (x P) partials, latency-bound otherwise
template <int D = 8, class F>
__device__ __forceinline__ double ordered_sum(int n, F&& v) {
  double acc = 0.0;
  int j = 0;
  for (; j + D <= n; j += D) {
    double t[D];
#pragma unroll
    for (int u = 0; u < D; ++u) t[u] = v(j + u);
#pragma unroll
    for (int u = 0; u < D; ++u) acc += t[u];
  }
  if (j < n) {   // the tail as one predicated batch (a rolled load-add loop waits for each load in turn)
    double t[D];
#pragma unroll
    for (int u = 0; u < D; ++u) t[u] = j + u < n ? v(j + u) : 0.0;
#pragma unroll
    for (int u = 0; u < D; ++u)
      if (j + u < n) acc += t[u];
  }
  return acc;
}

// Partial sum of slot s for element (a, n): the slot's fp32 value, or with split parts (P > 1,
// common.cuh split_parts) the fp64 sum of its P parts in part order.
__device__ __forceinline__ double slot_part(const SlotPartials& Gp, int P, int s, int64_t cap, int ldg, int a, int n) {
  if (P > 1) {
    const float* g = Gp.sub + (((int64_t)s * kSplitMax) * Gp.sub_cap + a) * ldg + n;
    const int64_t qs = Gp.sub_cap * ldg;
    float t[kSplitMax];
#pragma unroll
    for (int q = 0; q < kSplitMax; ++q) t[q] = q < P ? __ldg(g + q * qs) : 0.f;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < kSplitMax; ++q)
      if (q < P) acc += (double)t[q];
    return acc;
  }
  if (Gp.f32) return (double)__ldg((const float*)Gp.p + ((int64_t)s * cap + a) * ldg + n);
  return __ldg((const double*)Gp.p + ((int64_t)s * cap + a) * ldg + n);
}

__device__ __forceinline__ int parts_of(const SlotPartials& Gp, int S) {
  return (Gp.f32 && Gp.sub) ? split_parts(Gp.cnt_g ? Gp.cnt_g[0] : Gp.L_g_host, S) : 1;
}

// sum over slots (fixed slot order) of the slot partial sums: the definition every consumer of
// the slot partials shares (epilogue, k_slot_reduce), so a row's G is the same whichever runs it
// D: loads in flight per call (callers with many coordinates per lane: fewer).  KIND: 0 = the
// partials' type read at run time, 1 = fp64 partials, 2 = fp32 partials (with split parts): a
// caller that knows the type compiles one branch (kernel code size: latency of short kernels)
template <int D = 8, int KIND = 0>
__device__ __forceinline__ double slot_sum(SlotPartials Gp, int S, int64_t cap, int ldg, int a, int n) {
  if (KIND == 1) {
    const double* g = (const double*)Gp.p + (int64_t)a * ldg + n;
    const int64_t st = cap * ldg;
    return ordered_sum<D>(S, [&](int s) { return g[s * st]; });
  }
  const int P = parts_of(Gp, S);
  // split parts: each slot's value already sums up to 8 partials (loads in flight); rolled loop
  if (P > 1) return ordered_sum<(D >= 16 ? 4 : 2)>(S, [&](int s) { return slot_part(Gp, P, s, cap, ldg, a, n); });
  // one partial per slot (the common case; the loop the whole-L epilogue streams at HBM rate)
  if (KIND == 2 || Gp.f32) {
    const float* g = (const float*)Gp.p + (int64_t)a * ldg + n;
    const int64_t st = cap * ldg;
    return ordered_sum<D>(S, [&](int s) { return (double)g[s * st]; });
  }
  const double* g = (const double*)Gp.p + (int64_t)a * ldg + n;
  const int64_t st = cap * ldg;
  return ordered_sum<D>(S, [&](int s) { return g[s * st]; });
}

// slot_sum kept out of line: in the few-row update the split-part / fp64-partial branch is the
// cold one, and its unrolled loads would sit in the middle of the hot path's instruction stream
template <int D, int KIND>
__device__ __noinline__ double slot_sum_outlined(SlotPartials Gp, int S, int64_t cap, int ldg, int a, int n) {
  return slot_sum<D, KIND>(Gp, S, cap, ldg, a, n);
}

// coordinate n of the point the contraction used for candidate l (master value w64 if none)
__device__ __forceinline__ double eval_coord(const EvalPoint& ev, int l, int n, double w64) {
  int64_t i = (int64_t)l * ev.ld + n;
  if (ev.hi) return ((double)__half2float(ev.hi[i]) + (ev.lo ? (double)__half2float(ev.lo[i]) : 0.0)) * 0.0625;
  if (ev.f32) return (double)ev.f32[i];
  return w64;
}

// Split fp16 operand of one coordinate: w is scaled by 2^4 (|w| <= 1 -> <= 16) so most w_lo stay
// normal fp16; hi = fp16(2^4 w), lo = fp16(2^4 w - hi) (fine rows; 0 for coarse rows).  hi + lo =
// 2^4 w to ~2^-22 relative (absolute error <= 3e-8 / 16 per coordinate from lo subnormals).
__device__ __forceinline__ void operand_f16x2_coord(double w, bool fine_row, __half* hi_out, __half* lo_out) {
  const double w16 = w * 16.0;
  const __half hi = __double2half(w16);
  *hi_out = hi;
  if (lo_out) *lo_out = fine_row ? __double2half(w16 - (double)__half2float(hi)) : __double2half(0.0);
}

// w_old and w_e of candidate l, coordinates lane + 32 v (loaded ahead of the slot sums)
template <int V>
__device__ __forceinline__ void load_row(const UpdateArgs& u, int l, int lane, double (&wo)[V], double (&we)[V]) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int n = lane + 32 * v;
    wo[v] = 0.0;
    we[v] = 0.0;
    if (n < u.N) {
      wo[v] = u.W64[(int64_t)l * u.N + n];
      we[v] = eval_coord(u.ev, l, n, wo[v]);
    }
  }
}

// K3 core for candidate l, G already summed over the slots (acc[v] = coordinate
// lane + 32 v): g = G / M - 3 w_e; g <- g - E g; w = g / ||g||; d = 1 - |w . w_old| as
// 0.5 ||w - s w_old||^2 (A1/A2); converged iff d <= tol.  w_e is the operand the contraction was
// evaluated at (the whole of eq. (5) at one point, so the map keeps its vanishing
// tangent Jacobian at the fixed points); w_old is the fp64 master row.  Writes the new master row
// and, for a row that stays active, its next operand row; returns keep (still active).
template <int V>
__device__ __forceinline__ bool epilogue_core(int l, int lane, const double (&acc)[V], double s4_slots,
                                              const double (&wo)[V], const double (&we)[V], const UpdateArgs& u,
                                              int k, int t) {
  const int N = u.N;
  double g[V];
  double s4g = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    int n = lane + 32 * v;
    s4g += we[v] * acc[v];
    g[v] = (n < N) ? acc[v] / u.M - 3.0 * we[v] : 0.0;     // PAPER.md:244-245 (eq. (5), A3)
  }
  // SIMT: sum y^4 from its slot partials; TC: the identity w . sum_m y^3 x = sum_m y^4 (approximate alpha)
  s4g = warp_sum(s4g);
  const double s4 = u.s4p ? s4_slots : s4g;
  project_warp<V>(g, u.Wacc, k, N, lane);
  double ss = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) ss += g[v] * g[v];
  double nrm = sqrt(warp_sum(ss));
  // a non-finite update (fp16 range failure, non-finite data) retires the row and is reported
  // (Promotion::nonfinite): it must neither keep iterating to the cap nor enter the argmax
  const bool bad = !isfinite(nrm);
  bool deg = bad || nrm < kDegenerateNorm;
  double dot = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    g[v] = deg ? 0.0 : g[v] / nrm;
    dot += g[v] * wo[v];
  }
  dot = warp_sum(dot);
  double sg = dot < 0.0 ? -1.0 : 1.0;
  double dd = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    double e = g[v] - sg * wo[v];
    dd += e * e;
  }
  dd = 0.5 * warp_sum(dd);
  const bool conv = !deg && dd <= u.tol;                    // PAPER.md:249-250 (A2)
  const bool keep = !deg && !conv;
  const Promotion& pr = u.pr;
  bool fine_row = pr.fine == nullptr;                       // (no promotion state: two-pass rows)
  if (pr.fine) {
    fine_row = pr.fine[l] != 0;
    // DESIGN.md §5 precision promotion (decided identically on every lane)
    if (keep && !fine_row && ((dd <= pr.d_promote && dd > pr.ratio * pr.dprev[l]) || t >= pr.t_force))
      fine_row = true;
  }
  if (!deg) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      int n = lane + 32 * v;
      if (n < N) u.W64[(int64_t)l * N + n] = g[v];
    }
  }
  if (keep) {   // next operand row of l (ld coordinates, zero padded); eval reads above came first
    const int ld = u.ev.ld;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int n = lane + 32 * v;
      if (n < ld) {
        const double w = n < N ? g[v] : 0.0;
        const int64_t i = (int64_t)l * ld + n;
        if (u.ev.hi)
          operand_f16x2_coord(w, fine_row, u.ev.hi + i, u.ev.lo ? u.ev.lo + i : nullptr);
        else if (u.ev.f32)
          u.ev.f32[i] = (float)w;
      }
    }
  }
  if (lane == 0) {
    if (bad && pr.nonfinite) atomicAdd(pr.nonfinite, 1);
    u.iters[l] = t;
    u.alpha_old[l] = s4 / u.M - 3.0;                        // eq. (2) at w_old (A15)
    u.state[l] = deg ? ST_DEGENERATE : (conv ? ST_CONVERGED : ST_ACTIVE);
    if (pr.fine && keep) {
      pr.fine[l] = fine_row ? 1 : 0;
      pr.dprev[l] = dd;
    }
  }
  return keep;
}

// Order-preserving compaction by one block (deterministic), stably partitioned into coarse rows
// followed by fine rows; act_in null: the identity list.  Each thread takes a contiguous run of
// positions; counts are scanned with warp shuffles and one warp over the warp totals.  Returns
// (n_coarse + n_fine, n_coarse) in every thread.  copy_dst (may be act_in): the list is written
// there too.
__device__ __forceinline__ int2 compact_block(const int* act_in, const uint8_t* __restrict__ keep,
                                              const uint8_t* __restrict__ fine, int L_in, int* act_out,
                                              int* copy_dst = nullptr) {
  __shared__ int wc[32], wf[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = (blockDim.x + 31) >> 5;
  const int per = (L_in + blockDim.x - 1) / blockDim.x;
  const int b = t * per, e = min(L_in, b + per);
  // few positions per thread (the latency-bound lists): a thread's flags and ids are loaded together
  // and kept in registers for the second pass -- two load round trips instead of three per position
  // and pass; the list written is the same
  constexpr int R = 4;
  const bool few = per <= R;   // block-uniform
  int ids[R];
  bool kp[R], fn[R];
  int cc = 0, cf = 0;
  if (few) {
    uint8_t kq[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int a = b + r;
      kq[r] = a < e ? keep[a] : (uint8_t)0;
      ids[r] = a < e ? (act_in ? act_in[a] : a) : 0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      kp[r] = kq[r] != 0;
      fn[r] = kp[r] && fine && fine[ids[r]];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cc += (kp[r] && !fn[r]) ? 1 : 0;
      cf += fn[r] ? 1 : 0;
    }
  } else {
    for (int a = b; a < e; ++a) {
      if (!keep[a]) continue;
      int id = act_in ? act_in[a] : a;
      if (fine && fine[id]) ++cf; else ++cc;
    }
  }
  int ic = cc, jf = cf;   // inclusive warp scans of (cc, cf)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int vc = __shfl_up_sync(0xffffffffu, ic, o), vf = __shfl_up_sync(0xffffffffu, jf, o);
    if (lane >= o) {
      ic += vc;
      jf += vf;
    }
  }
  if (lane == 31) {
    wc[w] = ic;
    wf[w] = jf;
  }
  __syncthreads();
  if (w == 0) {   // inclusive scan of the warp totals
    int xc = lane < nw ? wc[lane] : 0, xf = lane < nw ? wf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int vc = __shfl_up_sync(0xffffffffu, xc, o), vf = __shfl_up_sync(0xffffffffu, xf, o);
      if (lane >= o) {
        xc += vc;
        xf += vf;
      }
    }
    wc[lane] = xc;
    wf[lane] = xf;
  }
  __syncthreads();
  const int n_coarse = wc[nw - 1], n_fine = wf[nw - 1];
  const int base_c = (w ? wc[w - 1] : 0) + ic - cc, base_f = (w ? wf[w - 1] : 0) + jf - cf;
  int pc = base_c, pf = n_coarse + base_f;
  if (few) {   // (every thread read its act_in entries before the barriers above: copy_dst may be act_in)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (kp[r]) {
        const int p = fn[r] ? pf++ : pc++;
        act_out[p] = ids[r];
        if (copy_dst) copy_dst[p] = ids[r];
      }
    }
  } else {
    for (int a = b; a < e; ++a) {
      if (!keep[a]) continue;
      int id = act_in ? act_in[a] : a;
      if (fine && fine[id]) act_out[pf++] = id; else act_out[pc++] = id;
    }
  }
  __syncthreads();   // wc / wf are read above by every thread
  if (!few && copy_dst)
    for (int j = t; j < n_coarse + n_fine; j += blockDim.x) copy_dst[j] = act_out[j];
  return make_int2(n_coarse + n_fine, n_coarse);
}

// End of an iteration (one thread): counts, history, iteration state, loop condition.
__device__ __forceinline__ void finish_iteration(const UpdateArgs& u, int2 r, int L_in, int t) {
#ifdef OICA_DEBUG_CHECKS
  if (r.x < 0 || r.x > L_in || r.y < 0 || r.y > r.x || t < 1 || (u.K_loop > 0 && t > u.K_loop + 1)) {
    printf("oica debug: iteration %d: compaction kept %d (coarse %d) of %d rows\n", t, r.x, r.y, L_in);
    __trap();
  }
#endif
  u.cnt_out[0] = r.x;
  u.cnt_out[1] = r.y;
  if (u.host_mapped) {
    ((volatile int*)u.host_mapped)[0] = r.x;
    ((volatile int*)u.host_mapped)[1] = r.y;
  }
  u.ctl->done = 0u;
  if (L_in > 0) {   // an executed iteration (a host-launched batch may enqueue a few beyond the last)
    if (u.hist) {
      u.hist[2 * t] = r.x;
      u.hist[2 * t + 1] = r.y;
    }
    u.ctl->t = t + 1;
    u.ctl->sum_active += L_in;
  }
  // do ... while (t < K and B != {})
  const int t_next = L_in > 0 ? t + 1 : t;
  const bool more = r.x > 0 && t_next <= u.K_loop;
  const bool run = L_in > 0 && more && r.x > u.loop_thr;
  if (u.loop) cudaGraphSetConditional(u.loop, run ? 1u : 0u);
  if (u.gate_out) {
    u.gate_out[0] = run ? r.x : 0;
    u.gate_out[1] = run ? r.y : 0;
  }
  if (u.loop_next) cudaGraphSetConditional(u.loop_next, more ? 1u : 0u);
}


// One pass of the few-row update over rows a_base + rb, rb < RPB (the block's warps: RPB rows x NG
// warps; every thread of the block must call it): the NG warps of a row sum its slot partials, 32
// coordinates each, in fixed slot order; the row's first warp runs epilogue_core.  keep_sh[rb] =
// the row stays active (and keep[a] when write_keep).
template <int NG, bool F32, int RPB>
__device__ __forceinline__ void update_pass(const UpdateArgs& u, int a_base, int L_in, int t, int k,
                                            double (*gsh)[NG * 32], double* s4sh, int* keep_sh, bool write_keep,
                                            long long* stamp = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = warp / NG, grp = warp - rb * NG;
  const int a = a_base + rb;
  const bool row_ok = rb < RPB && a < L_in;
  int l = 0;
  double wo[NG], we[NG];
  if (row_ok) {
    l = u.act_in[a];
#ifdef OICA_DEBUG_CHECKS
    if (l < 0 || l >= u.cap || L_in > u.L_ub) {
      printf("oica debug: update row %d -> candidate %d (cap %lld, L_in %d, L_ub %d)\n", a, l, (long long)u.cap,
             L_in, u.L_ub);
      __trap();
    }
#endif
    const int n = grp * 32 + lane;
    // (D partials in flight per lane: with few active rows the slot chain is latency-bound; the
    // association is the same sequential slot order whatever the depth)
    constexpr int D = NG >= 8 ? 8 : (NG == 1 ? 32 : 16);
    if (F32 && parts_of(u.G, u.S) == 1) {
      // one fp32 partial per slot: the first D slot loads (addresses from the row position a alone)
      // are issued before the row's w_old / w_e loads, which wait for act_in[a] -- one L2 round
      // trip for both instead of a chain (slot_sum's sum: acc = 0, += slot 0, 1, ... in order)
      const float* g = (const float*)u.G.p + (int64_t)a * u.ldg + n;
      const int64_t st = u.cap * u.ldg;
      const bool nk = n < u.N;
      float tb[D];
#pragma unroll
      for (int q = 0; q < D; ++q) tb[q] = (nk && q < u.S) ? g[q * st] : 0.f;
      if (grp == 0) load_row<NG>(u, l, lane, wo, we);
      if (stamp) stamp[0] = clock64() + (long long)(wo[0] * 0.0);   // (experiments build: after the row loads landed)
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < D; ++q)
        if (q < u.S) acc += (double)tb[q];
      for (int j = D; j < u.S; j += D) {
#pragma unroll
        for (int q = 0; q < D; ++q) tb[q] = (nk && j + q < u.S) ? g[(int64_t)(j + q) * st] : 0.f;
#pragma unroll
        for (int q = 0; q < D; ++q)
          if (j + q < u.S) acc += (double)tb[q];
      }
      gsh[rb][n] = nk ? acc : 0.0;
    } else {
      if (grp == 0) load_row<NG>(u, l, lane, wo, we);   // (in flight with the slot sums below)
      // F32: only the split-part case gets here (the cold branch, out of line); fp64 partials (the
      // FP32 step): this IS the row's slot sum, inline
      if (F32)
        gsh[rb][n] = n < u.N ? slot_sum_outlined<D, 2>(u.G, u.S, u.cap, u.ldg, a, n) : 0.0;
      else
        gsh[rb][n] = n < u.N ? slot_sum<D, 1>(u.G, u.S, u.cap, u.ldg, a, n) : 0.0;
    }
    if (grp == 0 && lane == 0 && u.s4p)
      s4sh[rb] = ordered_sum<16>(u.S, [&](int s) { return __ldg(u.s4p + (int64_t)s * u.cap + a); });
  }
  if (stamp) stamp[1] = clock64();
  __syncthreads();
  if (stamp) stamp[2] = clock64();
  if (row_ok && grp == 0) {
    double acc[NG];
#pragma unroll
    for (int v = 0; v < NG; ++v) acc[v] = gsh[rb][lane + 32 * v];
    const bool kp = epilogue_core<NG>(l, lane, acc, u.s4p ? s4sh[rb] : 0.0, wo, we, u, k, t);
    if (lane == 0) {
      keep_sh[rb] = kp ? 1 : 0;
      if (write_keep) u.keep[a] = kp ? 1 : 0;
    }
  }
}

// One row a of the few-row update with the whole block on its slot partials (S * NP * 8 bytes of
// shared memory T): the warps load the S slots' values of the row into T in parallel (slot_part:
// the fp64 or fp32 partial, or the fp64 sum of a slot's split parts in part order), then warp g
// sums coordinates g*32 + lane over the slots in slot order from T -- the same sequential
// association as slot_sum -- and warp 0 runs epilogue_core.  Every thread of the block must call
// it.  keep[a] is written.
// S4SH (the persistent FP32 loop): the row's sum-y^4 slot partials are loaded with the G partials,
// in parallel, into T[S * NP ...] (S more doubles of shared memory) and summed from there in slot
// order -- one L2 round trip instead of a chain of S / 16 (Exp. 1: see DESIGN.md §5)
template <int NG, bool S4SH = false>
__device__ __forceinline__ void update_row_coop(const UpdateArgs& u, int a, int L_in, int t, int k, double* T,
                                                double (*gsh)[NG * 32], double* s4sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int NPd = NG * 32;
  const int P = parts_of(u.G, u.S);
  int l = 0;
  double wo[NG], we[NG];
  if (a < L_in) {
    l = u.act_in[a];
    if (warp == 0) load_row<NG>(u, l, lane, wo, we);
    if (S4SH) {
      // a warp's slots (S / 8 of them at Exp. 1's S = 78) loaded into registers together, then
      // stored: a load-store loop through the generic T pointer waits for each load in turn
      constexpr int B = 8;
      for (int s0 = warp; s0 < u.S; s0 += nw * B) {
        double v[B][NG];
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const int s = s0 + b * nw;
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            const int n = g * 32 + lane;
            v[b][g] = (s < u.S && n < u.N) ? slot_part(u.G, P, s, u.cap, u.ldg, a, n) : 0.0;
          }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const int s = s0 + b * nw;
          if (s < u.S)
#pragma unroll
            for (int g = 0; g < NG; ++g) T[s * NPd + g * 32 + lane] = v[b][g];
        }
      }
    } else {
      for (int s = warp; s < u.S; s += nw) {
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const int n = g * 32 + lane;
          T[s * NPd + n] = n < u.N ? slot_part(u.G, P, s, u.cap, u.ldg, a, n) : 0.0;
        }
      }
    }
    if (S4SH && u.s4p)
      for (int s = threadIdx.x; s < u.S; s += blockDim.x) T[u.S * NPd + s] = __ldg(u.s4p + (int64_t)s * u.cap + a);
  }
  __syncthreads();
  if (a < L_in) {
    if (warp < NG) {
      const int n = warp * 32 + lane;
      double acc = 0.0;
      for (int s = 0; s < u.S; ++s) acc += T[s * NPd + n];   // slot order (slot_sum's association)
      gsh[0][n] = acc;
    }
    if (warp == NG && lane == 0 && u.s4p) {
      if (S4SH) {
        double acc = 0.0;
        for (int s = 0; s < u.S; ++s) acc += T[u.S * NPd + s];   // slot order (ordered_sum's association)
        s4sh[0] = acc;
      } else {
        s4sh[0] = ordered_sum<16>(u.S, [&](int s) { return __ldg(u.s4p + (int64_t)s * u.cap + a); });
      }
    }
  }
  __syncthreads();
  if (a < L_in && warp == 0) {
    double acc[NG];
#pragma unroll
    for (int v = 0; v < NG; ++v) acc[v] = gsh[0][lane + 32 * v];
    const bool kp = epilogue_core<NG>(l, lane, acc, u.s4p ? s4sh[0] : 0.0, wo, we, u, k, t);
    if (lane == 0) u.keep[a] = kp ? 1 : 0;
  }
  __syncthreads();   // T / gsh are rewritten by the block's next row
}

}  // namespace upd
}  // namespace oica
