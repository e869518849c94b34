// K2a: fused GEMM-cube-GEMM on tcgen05 tensor cores (sm_100a), Y never leaves the SM.
//
// For one work unit = (128-row tile of active candidates, split-M slot s [, part of P when few
// rows remain: the slot's chunks divided among P CTAs, each with its own fp32 partial, P from
// the global active count only — common.cuh split_parts]) the CTA computes
//   Y   = W X_chunk                 GEMM1  (eq. (4))   -> TMEM, fp32
//   Y3  = y o y o y                  epilogue warps, fp16 A operand written back into TMEM
//   G  += Y3 X_chunk^T               GEMM2  (eq. (5))   -> TMEM, fp32 accumulator
// streaming X through shared memory in TMA-loaded chunks, and finally stores G (x 2^12) as the
// unit's fp32 slot partial Gp[s][row][n] (Gsub for parts).  No atomics: each unit owns its region, so the
// result of a row is independent of the tile it shares (bitwise-deterministic).
//
// Arithmetic (DESIGN.md §5 "precision"): X is rounded once to fp16 (11-bit significand, same
// as TF32).  The operand row is w_h = fp16(2^4 w) (one GEMM1 pass) or, for "fine" rows, w_h + w_l
// with w_l = fp16(2^4 w - w_h) (two passes, w to ~2^-22); fine tiles also run GEMM2 twice, on
// y^3 2^-6 rounded to fp16 and on its fp16 residual (y^3 to ~2^-22).  Fine rows are grouped at the end of
// the active list; tiles >= n_coarse/128 run the second passes (a coarse row in such a tile carries
// w_l = 0 and a zero y^3 residual, which add exact zeros: a row's result never depends on the
// rows it shares a tile with, so L-shard results are identical for any GPU count).  K3 evaluates the -3w term of eq. (5) at the SAME operand
// (consistent evaluation of the fixed-point map at the rounded point, whose tangent Jacobian
// vanishes at a fixed point).  y^3 2^-6 is rounded to fp16 for GEMM2 (1 pass).  Accumulation
// fp32 in TMEM per slot (stored as exact fp32 x 2^12), fp64 across slots (K3).  Issued tensor
// work = 2 (coarse tile) or 4 (fine tile) fp16 passes per 2 algorithmic GEMMs.
//
// Layout (NP <= 128, MT = 128):  TMEM  [W_hi NP/2 | (W_lo NP/2) | G NP | Y0 128 | Y1 128]
//                                 SMEM  X stages [NP][128] fp16, 128B-swizzled (2 TMA boxes)
//   (variant RG = 0: 4 Y slots of 64 samples, [NP][64] stages; kept for A/B timing)
// Layout (NP <= 64, MT = 64, release): TMEM [W_hi | (W_lo) | G | Y0 64 | Y1 64] in a 256-column
//   allocation, [NP][64] stages, ~70 KB of SMEM: two CTAs per SM.
// Every layout computes bitwise the same partials: split parts cut slots at multiples of 384
// samples (whole chunks of every width), and a fine tile's GEMM2 runs its y^3 and residual
// passes per 64-sample group, so the fp32 accumulation order does not depend on the chunk width.
// Layout (NP > 128, MT = 64):    TMEM  [W_hi <=128 | G NP | Y0 64 | Y1 64]
//                                 SMEM  (W_lo [128][NP], K-major SW128 boxes) + X stages [NP][64]
// (W_lo parts only in the LO-capable instantiation, launched when the list has fine rows.)
// GEMM1 runs R-1 chunks ahead of GEMM2 (R = number of Y slots), so the tensor pipe has
// (R-1) GEMM1s queued while the epilogue cubes a chunk.
// Y3 is written in place per 32-column group g: y^3 of columns [32g, 32g+32) as fp16 pairs in
// columns [32g, 32g+16), so the GEMM2 A-operand K-slice kk sits at column 32(kk/2) + 8(kk%2).
// Warp roles: 0 = TMA producer + TMEM allocator, 1 = MMA issuer (one elected lane), 2..5 =
// epilogue (warp w reaches TMEM lanes 32*(w%4)..+31 = rows of the tile).
//
// Cluster multicast (CL = 2, default for NP > 64 unless one row tile remains; an empty partner
// tile only streams its share and issues no MMA): the two CTAs of a cluster are two row tiles
// of the same slot, so they stream the same X chunks; each loads half the rows of every chunk
// and multicasts it to both (one L2 read feeds two SMs), and a stage is refilled only after
// both CTAs' MMAs released it (the `empty` barrier counts CL commits, multicast by every CTA).
// Measured (scripts/tc_variants.py, cfg-4 shape): the X stream alone takes 175 ms per full-L
// launch without multicast (L2 -> SM at ~6 TB/s paces the kernel) and 95 ms with CL = 2.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "kernels.cuh"

namespace oica {
namespace {

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifdef OICA_DEBUG_CHECKS
// debug build (build.py --debug-checks): a bounded wait -- a phase that never completes (a lost
// arrival, a wrong parity) traps instead of hanging the GPU; ~2^26 polls of <= 10 ms suspend hint
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t polls = 0;; ++polls) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
    if (done) return;
    if (polls > (1u << 26)) {
      printf("oica debug: mbarrier wait timed out (block %d thread %d parity %u)\n", blockIdx.x, threadIdx.x, parity);
      __trap();
    }
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// multicast variant: the box lands at the same smem offset in every CTA of ctaMask, and each
// destination CTA's mbarrier (same offset) receives the complete_tx of the bytes written there
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// (a0^3, a1^3) with packed fp32x2 multiplies (FMUL2): (a*a)*a per lane, exactly as two scalar
// FMULs would round it
__device__ __forceinline__ float2 cube2(uint32_t a0, uint32_t a1) {
  const unsigned long long av = ((unsigned long long)a1 << 32) | a0;
  unsigned long long sq, cu;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(sq) : "l"(av), "l"(av));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(cu) : "l"(sq), "l"(av));
  return make_float2(__uint_as_float((uint32_t)cu), __uint_as_float((uint32_t)(cu >> 32)));
}

// 8 consecutive floats (32-byte aligned) in one 256-bit store (sm_100)
__device__ __forceinline__ void st_v8(float* p, const float (&g)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(g[0]), "f"(g[1]), "f"(g[2]), "f"(g[3]),
               "f"(g[4]), "f"(g[5]), "f"(g[6]), "f"(g[7])
               : "memory");
}
__device__ __forceinline__ void st_v8_cs(float* p, const float (&g)[8]) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(g[0]), "f"(g[1]), "f"(g[2]),
               "f"(g[3]), "f"(g[4]), "f"(g[5]), "f"(g[6]), "f"(g[7])
               : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, %1;\n\t"
      "@px mov.s32 %0, 1;\n\t}"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// arrive on the mbarrier at the same smem offset in every CTA of ctaMask once prior MMAs complete
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc]
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

#define OICA_R8(i) "=r"(v[i + 0]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
#define OICA_W8(i) "r"(v[i + 0]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3]), "r"(v[i + 4]), "r"(v[i + 5]), "r"(v[i + 6]), "r"(v[i + 7])

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets lane (base+i), columns c..c+31
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : OICA_R8(0), OICA_R8(8), OICA_R8(16), OICA_R8(24)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), OICA_W8(0)
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      OICA_W8(0), OICA_W8(8)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ descriptors
// shared-memory matrix descriptor (tcgen05): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 [46,48), layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor, kind::f16: F16 x F16 -> F32, M = 128
__host__ __device__ constexpr uint32_t idesc_f16(int N, int b_mn_major) {
  return (1u << 4) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// SPLIT = LO-capable layout.  RG = Y-ring variant: 0 = default (narrow: 4 slots of 64 samples,
// wide: 2 slots of 64), 1 = narrow with 2 slots of 128 (the previous layout, for A/B timing).
template <int NP, bool SPLIT, int RG = 0>
struct Cfg {
  static constexpr bool WIDE = NP > 128;                         // wide layout (W_lo in SMEM)
  static constexpr bool WLO_TMEM = SPLIT && !WIDE;               // W_lo as a TMEM A operand
  static constexpr bool WLO_SMEM = SPLIT && WIDE;                // W_lo as an SMEM A operand
  // RG = 3 (NP <= 64): 2 slots of 192 samples -- more tensor work per chunk hand-off where the
  // narrow MMAs are short (the hand-offs, not the MMAs, pace small NP)
  // RG = 7 (NP <= 64): 2 slots of 64 samples in a 256-column TMEM allocation and ~70 KB of
  // shared memory, so TWO CTAs share an SM (two hand-off chains interleave on the tensor pipe)
  static constexpr int MT = WIDE ? 64 : RG == 1 ? 128 : RG == 3 ? 192 : 64;   // samples per chunk (GEMM1 N)
  // epilogue warps (one per TMEM lane quadrant; the kernel also runs with two per quadrant, each
  // taking every other 32-column group)
  static constexpr int NW = 4;   // (8 for the small-NP layout measured no faster: cfg 2 step 875 vs 881 TFLOP/s)
  static constexpr int THREADS = 64 + 32 * NW;
  static constexpr int R = (!WIDE && RG == 0) ? 4 : 2;           // Y slots in TMEM (GEMM1 look-ahead R-1)
  static constexpr int XB = NP * 128;                            // bytes of one [NP][64] swizzled box
  static constexpr int X_STAGE = NP * MT * 2;                    // bytes per X stage
  static constexpr int WLO_BOXES = (NP + 63) / 64;               // 64-column K-major boxes of W_lo
  static constexpr int WLO_BYTES = WLO_SMEM ? 128 * WLO_BOXES * 128 : 0;
  static constexpr int X_BUDGET = WLO_SMEM ? 131072 : 196608;
  static constexpr int STAGES = X_BUDGET / X_STAGE >= 8 ? 8 : X_BUDGET / X_STAGE;
  static constexpr int C_WHI = 0;
  static constexpr int C_WLO = NP / 2;                           // WLO_TMEM only
  static constexpr int C_G = WLO_TMEM ? NP : (WIDE ? 128 : NP / 2);
  static constexpr int C_Y0 = C_G + NP;                          // slot b at C_Y0 + b * MT
  static_assert(C_Y0 + R * MT <= 512, "TMEM budget");
  static constexpr int TCOLS = RG == 7 ? 256 : 512;             // TMEM columns allocated
  static_assert(C_Y0 + R * MT <= TCOLS, "TMEM allocation");
  static constexpr int SMEM = 1024 + WLO_BYTES + STAGES * X_STAGE + 1024;
  static constexpr int MINB = RG == 7 ? 2 : 1;                   // CTAs per SM
  static_assert(MINB == 1 || SMEM * MINB <= 227 * 1024, "shared memory for MINB CTAs per SM");
};

// CL = cluster size sharing each X chunk (multicast); RG = Y-ring variant (Cfg)
template <int NP, bool SPLIT, int EPI, int CL, int RG>
__global__ void __launch_bounds__(Cfg<NP, SPLIT, RG>::THREADS, Cfg<NP, SPLIT, RG>::MINB)
k_step_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWlo,
          const __half* __restrict__ Whi, const __half* __restrict__ Wlo, const int* __restrict__ act, int L_ub,
          int64_t M, int64_t slot_len,
          float* __restrict__ Gp, int64_t cap, int n_coarse_h, int S_, const int* __restrict__ cnt, int s_base,
          int S_total, float* __restrict__ Gsub, int64_t sub_cap, const int* __restrict__ cnt_g, int split,
          const int8_t* __restrict__ xshift) {
  constexpr int NW = Cfg<NP, SPLIT, RG>::NW;   // epilogue warps
  using C = Cfg<NP, SPLIT, RG>;
  constexpr int MT = C::MT;
  // MODE 0 = the step; timing experiments (scripts/tc_variants.py): 3 = no
  // epilogue (MMA + data), 4 = GEMM1 only, 5 = GEMM2 only, 6 = no MMA (X streaming only),
  // 7 = GEMM1 only with an fp16 accumulator, 8 = step with an fp16 GEMM1 accumulator read as the
  // low half of each 32-bit TMEM cell (probe of the 16-bit accumulator layout), 9 = step without
  // the X stream (stale stages), 10 = MMAs only (no X stream, no epilogue)
  constexpr int MODE = EPI;
  constexpr int EPI_ARRIVALS = 32 * NW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* s_wlo = smem;
  uint8_t* s_x = smem + C::WLO_BYTES;
  uint64_t* bars = (uint64_t*)(s_x + C::STAGES * C::X_STAGE);
  uint64_t* full = bars;                     // [STAGES]
  uint64_t* empty = full + C::STAGES;        // [STAGES]
  uint64_t* wlo_full = empty + C::STAGES;    // 1
  uint64_t* w_ready = wlo_full + 1;          // 1
  uint64_t* yfull = w_ready + 1;             // [R]
  uint64_t* y3ready = yfull + 4;             // [R]
  uint64_t* gdone = y3ready + 4;             // 1
  uint32_t* tmem_slot = (uint32_t*)(gdone + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // active-row count and coarse/fine split: from the device counters when the grid was sized
  // from an upper bound (iterations enqueued without a host round trip)
  const int L_act = cnt ? min(L_ub, cnt[0]) : L_ub;
  const int n_coarse = cnt ? cnt[1] : n_coarse_h;
  const int tile_lo0 = n_coarse / 128;
  if (L_act <= 0) return;   // grid-uniform
  // work unit (row tile, slot s of [s_base, s_base + S_), part of P): the grid was sized for the
  // largest tiles x P the device counts can ask for; P = split_parts of the global count
  // (common.cuh) divides a slot's chunks among P CTAs when few row tiles are active
  const int P = split ? split_parts(cnt_g ? cnt_g[0] : L_ub, S_total) : 1;
  const int n_t = (int)round_up(ceil_div(L_act, 128), CL);
  const int tile = (int)(blockIdx.x % n_t), rest = (int)(blockIdx.x / n_t);
  const int s = s_base + rest / P, part = rest % P;
  if (s >= s_base + S_) return;                      // cluster-uniform (n_t is a multiple of CL)
  if ((tile - tile % CL) * 128 >= L_act) return;   // cluster-uniform: no barrier was touched
  const int row0 = tile * 128;
  const int64_t m_slot = (int64_t)s * slot_len;
  // parts split the slot at multiples of 384 samples (a multiple of every chunk width MT), so a
  // part's samples -- and every fp32 partial -- are the same whichever layout runs the step
  constexpr int kPartUnit = 384;
  static_assert(kPartUnit % MT == 0, "part boundaries must be whole chunks");
  const int len_slot = (int)(min(M, m_slot + slot_len) - m_slot);
  const int nch_slot = (len_slot + MT - 1) / MT;
  const int nu_slot = (len_slot + kPartUnit - 1) / kPartUnit;
  const int c_lo = nu_slot * part / P * (kPartUnit / MT);
  const int c_hi = part + 1 == P ? nch_slot : nu_slot * (part + 1) / P * (kPartUnit / MT);
  const int64_t m_begin = m_slot + (int64_t)c_lo * MT;
  const int nchunk = c_hi - c_lo;
  // idle: the empty partner tile of a cluster (rows >= L_act) only streams its share of the
  // multicast chunks; it issues no MMA (its commits still release the shared stages)
  const bool idle = row0 >= L_act;
  const bool lo_pass = SPLIT && tile >= tile_lo0 && !idle;   // CTA-uniform

  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
  static_assert(CL == 1 || (NP / CL) % 8 == 0, "multicast slices must be whole 8-row swizzle atoms");
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CL);   // released by the MMA commit of every CTA that shares the stage
    }
    mbar_init(wlo_full, 1);
    mbar_init(w_ready, EPI_ARRIVALS);
    for (int b = 0; b < C::R; ++b) {
      mbar_init(&yfull[b], 1);
      mbar_init(&y3ready[b], EPI_ARRIVALS);
    }
    mbar_init(gdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  if (CL > 1)
    cluster_sync_all();   // peers multicast into this CTA's barriers: all must be initialised
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      if (C::WLO_SMEM && lo_pass) {
        mbar_expect_tx(wlo_full, C::WLO_BYTES);
        for (int kb = 0; kb < C::WLO_BOXES; ++kb) tma_load_2d(s_wlo + kb * 16384, &tmWlo, wlo_full, kb * 64, row0);
      }
      // CL > 1: this CTA loads rows [crank*SR, (crank+1)*SR) of every chunk and multicasts them
      // to the whole cluster (all CTAs of a cluster share the slot, hence the chunks)
      constexpr int SR = NP / CL;
      const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
      for (int j = 0; j < nchunk; ++j) {
        int st = j % C::STAGES;
        if (j >= C::STAGES) mbar_wait(&empty[st], ((j / C::STAGES) - 1) & 1);
        int m0 = (int)(m_begin + (int64_t)j * MT);
        if (MODE == 9 || MODE == 10) {   // experiment: no X stream (MMAs / epilogue on stale stages)
          mbar_arrive(&full[st]);
          continue;
        }
        mbar_expect_tx(&full[st], C::X_STAGE);
        uint8_t* dst = s_x + st * C::X_STAGE;
        for (int h = 0; h < MT / 64; ++h) {
          if (CL == 1)
            tma_load_2d(dst + h * C::XB, &tmX, &full[st], m0 + 64 * h, 0);
          else
            tma_load_2d_mc(dst + h * C::XB + crank * SR * 128, &tmX, &full[st], m0 + 64 * h, crank * SR, kMask);
        }
      }
      if (CL > 1)   // peers' releases of the last stages must land before this CTA may exit
        for (int j = nchunk > C::STAGES ? nchunk - C::STAGES : 0; j < nchunk; ++j)
          mbar_wait(&empty[j % C::STAGES], (j / C::STAGES) & 1);
    }
  } else if (warp == 1) {
    // ===== MMA issuer: the whole warp follows the schedule, one elected lane issues =====
    // (warp-uniform operands keep the descriptors in uniform registers: one UTCHMMA + an
    // add per MMA, no per-instruction lane waterfall)
    // GEMM1: B = X, MN-major (m contiguous); experiment MODE 7: fp16 accumulator (D format F16)
    constexpr uint32_t id1 = (MODE == 7 || MODE == 8) ? (idesc_f16(MT, 1) & ~(1u << 4)) : idesc_f16(MT, 1);
    constexpr uint32_t id2 = idesc_f16(NP, 0);   // GEMM2: B = X, K-major (K = m)
    const uint32_t t_g = tmem + C::C_G;
    const uint64_t dx0 = sdesc(smem_u32(s_x), C::XB, 1024);   // X as MN-major B (GEMM1)
    const uint64_t dk0 = sdesc(smem_u32(s_x), 16, 1024);      // X as K-major B (GEMM2)
    const uint64_t dw0 = sdesc(smem_u32(s_wlo), 16, 1024);    // W_lo as K-major A (variant B)
    mbar_wait(w_ready, 0);
    if (C::WLO_SMEM && lo_pass) mbar_wait(wlo_full, 0);
    tc_fence_after();
    auto gemm1 = [&](int j) {
      const int st = j % C::STAGES, b = j % C::R;
      mbar_wait(&full[st], (j / C::STAGES) & 1);
      tc_fence_after();
      if (MODE == 5 || MODE == 6 || idle) {   // idle tile; experiments: GEMM2 only / no MMA
        if (elect_one()) tc_commit(&yfull[b]);
        __syncwarp();
        return;
      }
      if (elect_one()) {
        const uint64_t bx = dx0 + (uint64_t)((st * C::X_STAGE) >> 4);
        const uint32_t t_y = tmem + C::C_Y0 + b * MT;
#pragma unroll
        for (int kb = 0; kb < NP / 16; ++kb)   // pass 1: W_hi (TMEM) x X
          mma_ts(t_y, tmem + C::C_WHI + kb * 8, bx + (uint64_t)(kb * 128), id1, kb > 0 ? 1u : 0u);
        if (lo_pass) {
#pragma unroll
          for (int kb = 0; kb < NP / 16; ++kb) {   // pass 2: W_lo x X
            if (C::WLO_TMEM)
              mma_ts(t_y, tmem + C::C_WLO + kb * 8, bx + (uint64_t)(kb * 128), id1, 1u);
            else
              mma_ss(t_y, dw0 + (uint64_t)(((kb >> 2) * 16384 + (kb & 3) * 32) >> 4), bx + (uint64_t)(kb * 128), id1,
                     1u);
          }
        }
        tc_commit(&yfull[b]);
      }
      __syncwarp();
    };
    auto gemm2 = [&](int j) {
      const int st = j % C::STAGES, b = j % C::R;
      mbar_wait(&y3ready[b], (j / C::R) & 1);
      tc_fence_after();
      if (MODE == 4 || MODE == 6 || MODE == 7 || idle) {   // idle tile; experiments: GEMM1 only / no MMA
        if (elect_one()) {
          if (CL > 1) tc_commit_mc(&empty[st], kMask); else tc_commit(&empty[st]);
        }
        __syncwarp();
        return;
      }
      if (elect_one()) {
        const uint64_t bk = dk0 + (uint64_t)((st * C::X_STAGE) >> 4);
        const uint32_t t_y3 = tmem + C::C_Y0 + b * MT;
        // per 64-sample group: the y^3 pass, then (fine tile) the pass on its fp16 residual
        // (columns 32g+16..) -- the accumulation order is then the same for every chunk width
#pragma unroll
        for (int g64 = 0; g64 < MT / 64; ++g64) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = 4 * g64 + k4;
            mma_ts(t_g, t_y3 + (kk >> 1) * 32 + (kk & 1) * 8,
                   bk + (uint64_t)(((kk >> 2) * C::XB + (kk & 3) * 32) >> 4), id2, (j > 0 || kk > 0) ? 1u : 0u);
          }
          if (lo_pass) {
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const int kk = 4 * g64 + k4;
              mma_ts(t_g, t_y3 + (kk >> 1) * 32 + 16 + (kk & 1) * 8,
                     bk + (uint64_t)(((kk >> 2) * C::XB + (kk & 3) * 32) >> 4), id2, 1u);
            }
          }
        }
        if (CL > 1)
          tc_commit_mc(&empty[st], kMask);
        else
          tc_commit(&empty[st]);
      }
      __syncwarp();
    };
    // GEMM1 runs R-1 chunks ahead of GEMM2: slot (j+R-1) % R was last read by GEMM2(j-1),
    // issued earlier on the in-order tensor pipe
    for (int j = 0; j < C::R - 1 && j < nchunk; ++j) gemm1(j);
    for (int j = 0; j < nchunk; ++j) {
      if (j + C::R - 1 < nchunk) gemm1(j + C::R - 1);
      gemm2(j);
    }
    if (elect_one()) tc_commit(gdone);
    __syncwarp();
  } else {
    // ===== epilogue warps (NW warps; warp w reaches TMEM lanes 32*(w%4)..+31 = tile rows; the
    // NW/4 warps of one lane quadrant split the columns in 32-column groups) =====
    constexpr int NH = NW / 4;
    const int q = warp & 3, h = (warp - 2) >> 2;
    // fp16 range of the GEMM2 operand (DESIGN.md §5 "range"): |y| <= ||x_m|| for a unit row, and
    // xshift[b] = dsh is the least shift with max ||x_m|| <= 2^(7+dsh) over the 384-sample block
    // b, so y^3 2^-6 2^(-3 dsh) < 2^15 never overflows fp16 (65504).  The CTA takes the largest
    // shift over its sample range; 0 (every shipped workload) is the unscaled arithmetic.
    int dsh = 0;
    if (xshift && nchunk > 0) {
      const int64_t b0 = m_begin / kShiftBlock, b1 = ceil_div(min(M, m_begin + (int64_t)nchunk * MT), kShiftBlock);
      int v = 0;
      for (int64_t b = b0 + lane; b < b1; b += 32) v = max(v, (int)__ldg(xshift + b));
      dsh = __reduce_max_sync(0xffffffffu, v);
    }
    const float csc = __int_as_float((127 - 3 * dsh) << 23);   // 2^(-3 dsh), exact scaling
    const float gsc = __int_as_float((127 + 12 + 3 * dsh) << 23);   // 2^(12 + 3 dsh): flush unscale
    const int r = q * 32 + lane;
    const int row = row0 + r;
    const bool coarse_row = row < n_coarse;   // (fine tiles only: rows before the coarse/fine boundary)
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // W operand rows -> TMEM (A operand of GEMM1, fp16 pairs per 32-bit column)
    {
      bool ok = row < L_act;
      const int64_t id = ok ? (int64_t)__ldg(act + row) : 0;   // operand rows are stored by candidate id
#ifdef OICA_DEBUG_CHECKS
      if (ok && (id < 0 || id >= cap)) {
        printf("oica debug: step row %d -> candidate %lld outside [0, %lld)\n", row, (long long)id, (long long)cap);
        __trap();
      }
#endif
      // 16-byte loads, up to 32 of them in flight per thread (one L2 round trip for NP <= 128)
      const uint4* wh = (const uint4*)(Whi + id * NP);
      const uint4* wl = (const uint4*)(Wlo + id * NP);
      constexpr int CB = NP / 2 < 64 ? NP / 2 : 64;   // 32-bit columns per batch (a multiple of 8)
#pragma unroll 1
      for (int c0 = CB * h; c0 < NP / 2; c0 += CB * NH) {
        uint4 a[CB / 4];
#pragma unroll
        for (int k = 0; k < CB / 4; ++k) a[k] = ok ? __ldg(wh + c0 / 4 + k) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int k = 0; k < CB / 8; ++k) {
          const uint32_t v[8] = {a[2 * k].x, a[2 * k].y, a[2 * k].z, a[2 * k].w,
                                 a[2 * k + 1].x, a[2 * k + 1].y, a[2 * k + 1].z, a[2 * k + 1].w};
          tmem_st8(tmem + lane_off + C::C_WHI + c0 + 8 * k, v);
        }
        if (C::WLO_TMEM && lo_pass) {
#pragma unroll
          for (int k = 0; k < CB / 4; ++k) a[k] = ok ? __ldg(wl + c0 / 4 + k) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int k = 0; k < CB / 8; ++k) {
            const uint32_t v[8] = {a[2 * k].x, a[2 * k].y, a[2 * k].z, a[2 * k].w,
                                   a[2 * k + 1].x, a[2 * k + 1].y, a[2 * k + 1].z, a[2 * k + 1].w};
            tmem_st8(tmem + lane_off + C::C_WLO + c0 + 8 * k, v);
          }
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(w_ready);
    }
    // Y group g = columns [32g, 32g+32) -> y^3 2^-6 as fp16 pairs in columns [32g, 32g+16)
    // (in place, inside the group this warp owns: the A operand K-slice kk of GEMM2 sits at
    // column 32*(kk/2) + 8*(kk%2))
    constexpr int NG = MT / 32 / NH;   // groups per warp
    for (int j = 0; j < nchunk; ++j) {
      const int b = j % C::R;
      const uint32_t t_y = tmem + lane_off + C::C_Y0 + b * MT;
      mbar_wait(&yfull[b], (j / C::R) & 1);
      tc_fence_after();
      if ((MODE >= 3 && MODE != 8 && MODE != 9) || idle) {   // idle tile; experiment: no TMEM traffic (MMA pipeline upper bound)
        tc_fence_before();
        mbar_arrive(&y3ready[b]);
        continue;
      }
      constexpr int GB = NG > 4 ? NG / 2 : NG;   // groups per TMEM-load batch (register budget)
#pragma unroll
      for (int g0 = 0; g0 < NG; g0 += GB) {
        uint32_t v[GB][32];
#pragma unroll
        for (int w = 0; w < GB; ++w) tmem_ld32(t_y + 32 * (h + NH * (g0 + w)), v[w]);
        tmem_wait_ld();
        // SC: the range shift is active (CTA-uniform branch outside the element loop: the common
        // dsh == 0 case runs exactly the unscaled instruction sequence)
        auto cube_groups = [&](auto SC) {
          constexpr bool scaled = decltype(SC)::value;
#pragma unroll
          for (int w = 0; w < GB; ++w) {
            const int u = g0 + w;
            uint32_t pk[16];
            if (SPLIT && lo_pass) {   // fine tile: also the fp16 residual y^3 2^-6 - hi (GEMM2 second pass)
              uint32_t pl[16];   // (zero for a coarse row sharing the tile: its result must not depend on its tile)
#pragma unroll
              for (int k = 0; k < 32; k += 2) {
                const float2 cc = cube2(v[w][k], v[w][k + 1]);
                const float c0 = scaled ? cc.x * csc : cc.x, c1 = scaled ? cc.y * csc : cc.y;
                __half2 hh = __floats2half2_rn(c0, c1);
                pk[k / 2] = *reinterpret_cast<uint32_t*>(&hh);
                float2 hf = __half22float2(hh);
                __half2 hl = __floats2half2_rn(c0 - hf.x, c1 - hf.y);
                pl[k / 2] = coarse_row ? 0u : *reinterpret_cast<uint32_t*>(&hl);
              }
              tmem_st16(t_y + 32 * (h + NH * u) + 16, pl);
            } else {
#pragma unroll
              for (int k = 0; k < 32; k += 2) {
                // accumulator = 2^4 y 2^-6 = y / 4 (W scaled by 2^4, X by 2^-6)  ->  acc^3 = 2^-6 y^3
                if (MODE == 8) {   // experiment: fp16 accumulator, read as the low half of each cell
                  v[w][k] = __float_as_uint(__half2float(__ushort_as_half((unsigned short)(v[w][k] & 0xffffu))));
                  v[w][k + 1] = __float_as_uint(__half2float(__ushort_as_half((unsigned short)(v[w][k + 1] & 0xffffu))));
                }
                const float2 cc = cube2(v[w][k], v[w][k + 1]);
                __half2 hh = scaled ? __floats2half2_rn(cc.x * csc, cc.y * csc) : __floats2half2_rn(cc.x, cc.y);
                pk[k / 2] = *reinterpret_cast<uint32_t*>(&hh);
              }
            }
            tmem_st16(t_y + 32 * (h + NH * u), pk);   // Y^3 (fp16 pairs): A operand of GEMM2
          }
        };
        if (dsh == 0)
          cube_groups(std::false_type{});
        else
          cube_groups(std::true_type{});
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&y3ready[b]);
    }
    // G (fp32, scaled 2^-12 2^(-3 dsh): y^3 by 2^-6 2^(-3 dsh), X by 2^-6) -> fp32 slot partial
    // (x 2^(12 + 3 dsh): exact)
    mbar_wait(gdone, 0);
    tc_fence_after();
    float* out = P > 1 ? Gsub + (((int64_t)s * kSplitMax + part) * sub_cap + row) * NP : Gp + ((int64_t)s * cap + row) * NP;
    bool ok = row < L_act && nchunk > 0;
#pragma unroll 1
    for (int c = 32 * h; c < NP && !idle; c += 32 * NH) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + C::C_G + c, v);
      tmem_wait_ld();
      if (ok) {
        // 32-byte vector stores (one full sector each: the thread's row is contiguous, the warp's
        // 32 rows are not, so scalar stores cost a partial-sector write per element -- measured
        // ~4 us per 128 x 64 partial, 20% of a cfg-2 unit).  Streaming (.cs: keep the X planes
        // in L2), except the few rows of split parts, which the update reads next.
#pragma unroll
        for (int k = 0; k < 32; k += 8)
          if (NP % 32 == 0 || c + k < NP) {   // (NP is a multiple of 16: groups of 8 are whole)
            float g[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) g[e] = __uint_as_float(v[k + e]) * gsc;
            if (P > 1)
              st_v8(out + c + k, g);
            else
              st_v8_cs(out + c + k, g);
          }
      }
    }
    if (row < L_act && nchunk == 0 && h == 0)
      for (int c = 0; c < NP; ++c) out[c] = 0.f;
  }
  tc_fence_before();
  if (CL > 1)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  if (!fn) throw Error(OICA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// current driver context (nullptr if unavailable): the launch attributes are per context
void cuda_current_context(CUcontext* out) {
  typedef CUresult (*GetCurFn)(CUcontext*);
  static GetCurFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuCtxGetCurrent", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) ? (GetCurFn)p : (GetCurFn)nullptr;
  }();
  *out = nullptr;
  if (fn) fn(out);
}

// 2D fp16 tensor [rows][cols] (row stride ld elements), box [box_rows][64], 128B swizzle
CUtensorMap make_map(const __half* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(OICA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int NP, bool SPLIT, int EPI, int CL, int RG>
void launch_cl(cudaStream_t st, const __half* Xh, int64_t ldx, int64_t M, const __half* Whi, const __half* Wlo,
               const int* act, int L_act, int64_t slot_len, int S, float* Gp, int64_t cap, int n_coarse, const int* cnt,
               const Upload& up, const SplitOut& so, const int8_t* xshift) {
  using C = Cfg<NP, SPLIT, RG>;
  auto kern = k_step_tc<NP, SPLIT, EPI, CL, RG>;
  // once per CUDA context the launch runs in (the step may also run in green contexts, runtime.cu)
  static CUcontext attr_ctx[4] = {};
  CUcontext cur = nullptr;
  cuda_current_context(&cur);
  bool known = false;
  for (CUcontext k : attr_ctx) known = known || (k == cur && cur != nullptr);
  if (!known) {
    OICA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    if (CL > 1) OICA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (CUcontext& k : attr_ctx)
      if (!k) {
        k = cur;
        break;
      }
  }
  CUtensorMap tx = make_map(Xh, NP, ldx, ldx, NP / CL);
  CUtensorMap tw = tx;
  if (C::WLO_SMEM) tw = make_map(Wlo, cap, NP, NP, 128);
  // a cluster = CL tiles of one slot (part); units per slot cover any device count <= L_act:
  // n_t <= n_tiles, and n_t P <= kSplitTarget / S whenever P > 1 (split_parts)
  int n_tiles = (int)round_up(ceil_div(L_act, 128), CL);
  if (so.enable) n_tiles = std::max<int>(n_tiles, (int)round_up(std::max(1, kSplitTarget / std::max(S, 1)), CL));
  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(C::THREADS);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  lc.gridDim = dim3((unsigned)(n_tiles * up.s_count));
  OICA_CUDA(cudaLaunchKernelEx(&lc, kern, tx, tw, Whi, Wlo, act, L_act, M, slot_len, Gp, cap, n_coarse, up.s_count, cnt,
                               up.s_base, S, so.sub, so.sub_cap, so.cnt_g, so.enable, xshift));
}

// Release build: the measured-best layout per NP --
//   NP <= 64        2 Y slots of 192 samples, no cluster (latency-bound chunk hand-offs); few
//                   units: 2 Y slots of 64 samples in 256 TMEM columns, two CTAs per SM;
//   64 < NP <= 128  2 Y slots of 128 samples, 2-CTA multicast clusters;
//   NP > 128        wide layout (2 Y slots of 64 samples), 2-CTA multicast clusters;
// one remaining row tile (the tail of a component) launches without a cluster partner, whose
// CTA would only stream its half of the chunks in step with the active one (same arithmetic).
// -DOICA_EXPERIMENTS adds the timing variants of profiles/r01/tc_experiments (OICA_TC_EPI
// modes 3-8 that skip work, OICA_TC_CL = 1|2|4 and OICA_TC_RING overrides); they are compiled
// out of the product library so no environment variable can change what the timed step does.
// NP <= 64: launches of at most this many (row tile, slot) units -- the tail of a component, small
// L (cfg 1) -- take the two-CTAs-per-SM layout (RG 7); more units the 192-sample layout (RG 3).
// Measured over eight components (scripts/ab_step.py, step TFLOP/s): cfg 1 80.8 (RG 3 always) ->
// 90.8; cfg 2 995 -> 1009; RG 7 for every launch: cfg 1 90.3, cfg 2 1021 eager but 2% slower in
// the device-side loop, and a full-L N = 32 launch 4% slower
constexpr int kRg7Units = 2 * 296;

template <int NP, bool SPLIT, int EPI>
void launch_variant(cudaStream_t st, const __half* Xh, int64_t ldx, int64_t M, const __half* Whi, const __half* Wlo,
                    const int* act, int L_act, int64_t slot_len, int S, float* Gp, int64_t cap, int n_coarse, const int* cnt,
                    const Upload& up, const SplitOut& so, const int8_t* xshift) {
  constexpr int CL2 = (NP / 2) % 8 == 0 ? 2 : 1;
  // release layout for this NP (bitwise the same arithmetic): NP <= 64 2 x 192-sample slots at
  // one CTA per SM for launches of more than kRg7Units (row tile, slot) units, else 2 x 64 at two
  // CTAs per SM; 64 < NP <= 128 2 x 128-sample slots; wide 2 x 64
  constexpr int RGN = NP <= 64 ? 7 : NP <= 128 ? 1 : 0;
#ifdef OICA_EXPERIMENTS
  static int cl_env = [] { const char* e = getenv("OICA_TC_CL"); return e ? atoi(e) : 0; }();
  static int ring = [] { const char* e = getenv("OICA_TC_RING"); return e ? atoi(e) : 0; }();
  const int cl = up.cl ? up.cl : cl_env ? cl_env : (NP > 64 && L_act > 128 ? 2 : 1);
  if constexpr (NP == 256) {   // 4-CTA multicast clusters
    if (cl == 4) {
      launch_cl<NP, SPLIT, EPI, 4, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
      return;
    }
  }
  if (NP <= 128 && ring == 4) {   // narrow 4 x 64-sample Y ring (measured slower)
    if (cl == 2)
      launch_cl<NP, SPLIT, EPI, CL2, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
    else
      launch_cl<NP, SPLIT, EPI, 1, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
    return;
  }
  if constexpr (NP <= 64) {   // two CTAs per SM (2 x 64-sample slots, 256 TMEM columns)
    if (ring == 24) {
      launch_cl<NP, SPLIT, EPI, 1, 7>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
      return;
    }
  }
  if (NP <= 64 && ring == 2) {   // small NP with 2 x 128-sample slots
    launch_cl<NP, SPLIT, EPI, 1, 1>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
    return;
  }
  static int rg7_units = [] { const char* e = getenv("OICA_TC_RG7_UNITS"); return e ? atoi(e) : kRg7Units; }();
#else
  const int cl = up.cl ? up.cl : (NP > 64 && L_act > 128 ? 2 : 1);
  constexpr int rg7_units = kRg7Units;
#endif
  if constexpr (NP <= 64) {
    // many work units (full L): 2 x 192-sample slots, one CTA per SM
    if ((int64_t)ceil_div(L_act, 128) * S > rg7_units) {
      launch_cl<NP, SPLIT, EPI, 1, 3>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
      return;
    }
  }
  if (NP > 64 && cl == 2)
    launch_cl<NP, SPLIT, EPI, CL2, RGN>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
  else
    launch_cl<NP, SPLIT, EPI, 1, RGN>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
}

template <int NP, bool SPLIT>
void launch_epi(cudaStream_t st, const __half* Xh, int64_t ldx, int64_t M, const __half* Whi, const __half* Wlo,
                const int* act, int L_act, int64_t slot_len, int S, float* Gp, int64_t cap, int t0, const int* cnt, const Upload& up, const SplitOut& so, const int8_t* xshift) {
#ifdef OICA_EXPERIMENTS
  static int epi = [] { const char* e = getenv("OICA_TC_EPI"); return e ? atoi(e) : 0; }();
  switch (epi) {
    case 3: launch_variant<NP, SPLIT, 3>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    case 4: launch_variant<NP, SPLIT, 4>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    case 5: launch_variant<NP, SPLIT, 5>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    case 6: launch_variant<NP, SPLIT, 6>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    case 7: launch_variant<NP, SPLIT, 7>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    case 8: launch_variant<NP, SPLIT, 8>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    case 9: launch_variant<NP, SPLIT, 9>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    case 10: launch_variant<NP, SPLIT, 10>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); return;
    default: break;
  }
#endif
  launch_variant<NP, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift);
}

template <bool SPLIT>
void launch_np(cudaStream_t st, const __half* Xh, int64_t ldx, int64_t M, int NP, const __half* Whi, const __half* Wlo,
               const int* act, int L_act, int64_t slot_len, int S, float* Gp, int64_t cap, int t0, const int* cnt, const Upload& up, const SplitOut& so, const int8_t* xshift) {
  switch (NP) {
    case 16: launch_variant<16, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 32: launch_variant<32, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 48: launch_variant<48, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 64: launch_epi<64, SPLIT>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 80: launch_variant<80, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 96: launch_variant<96, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 112: launch_variant<112, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 128: launch_epi<128, SPLIT>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 144: launch_variant<144, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 160: launch_variant<160, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 176: launch_variant<176, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 192: launch_variant<192, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 208: launch_variant<208, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 224: launch_variant<224, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 240: launch_variant<240, SPLIT, 0>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    case 256: launch_epi<256, SPLIT>(st, Xh, ldx, M, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, t0, cnt, up, so, xshift); break;
    default: throw Error(OICA_ERR_INVALID_ARGUMENT, "unsupported padded N for the tensor-core step");
  }
}

// fp16 plane row n = fp16(x_n 2^-6), zero padded to NP rows and ldx columns, for the columns
// [m_lo, m_hi) (multiples of 8).  One thread per 8 consecutive samples of a row (blockIdx.y =
// row): coalesced fp32 reads, one 16-byte store.
__global__ void k_x_prepare_f16(const float* __restrict__ X, int64_t ld, int N, int64_t M, int64_t ldx,
                                __half* __restrict__ Xh, int64_t m_lo, int64_t m_hi) {
  const int n = blockIdx.y;
  const int64_t m0 = m_lo + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (m0 >= m_hi) return;
  const float* x = X + (int64_t)n * ld;
  __align__(16) __half2 h[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t m = m0 + 2 * k;
    float a = (n < N && m < M) ? __ldg(x + m) : 0.f;
    float b = (n < N && m + 1 < M) ? __ldg(x + m + 1) : 0.f;
    h[k] = __floats2half2_rn(a * kXScale, b * kXScale);
  }
  *reinterpret_cast<uint4*>(Xh + (int64_t)n * ldx + m0) = *reinterpret_cast<uint4*>(h);
}

// xshift[b] for the 384-sample blocks b in [m_lo / 384, ceil(m_hi / 384)): the least dsh >= 0 with
// 1.01 max_m ||x_m|| <= 2^(7 + dsh) over the block's samples (DESIGN.md §5 "range"; capped at
// kMaxShift).  One CTA per block, one thread per sample.
__global__ void __launch_bounds__(kShiftBlock) k_block_shift(const float* __restrict__ X, int64_t ld, int N,
                                                             int64_t M, int64_t m_lo, int8_t* __restrict__ xshift) {
  __shared__ float red[kShiftBlock / 32];
  const int64_t b = m_lo / kShiftBlock + blockIdx.x;
  const int64_t m = b * kShiftBlock + threadIdx.x;
  float ss = 0.f;
  if (m < M)
    for (int n = 0; n < N; ++n) {
      const float x = __ldg(X + (int64_t)n * ld + m);
      ss = fmaf(x, x, ss);
    }
  // max over the block (ss >= 0: the float bit patterns order like the values)
  unsigned u = __reduce_max_sync(0xffffffffu, __float_as_uint(ss));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = __uint_as_float(u);
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.f;
    for (int w = 0; w < kShiftBlock / 32; ++w) mx = fmaxf(mx, red[w]);
    const float B = 1.01f * sqrtf(mx);
    int d = 0;
    while (d < kMaxShift && B > ldexpf(1.0f, 7 + d)) ++d;
    xshift[b] = (int8_t)d;
  }
}

}  // namespace

int launch_block_shift(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, int64_t m_lo, int64_t m_hi,
                       int8_t* xshift) {
  m_hi = std::min<int64_t>(m_hi, M);
  if (m_hi <= m_lo) return 0;
  const int64_t nb = ceil_div(m_hi, kShiftBlock) - m_lo / kShiftBlock;
  k_block_shift<<<(unsigned)nb, kShiftBlock, 0, st>>>(X, ld, N, M, m_lo, xshift);
  return 1;
}

bool tc_supported(int N) { return N >= 1 && N <= 256; }
int tc_np(int N) { return (int)round_up(N < 16 ? 16 : N, 16); }

int launch_step_tc(cudaStream_t st, const __half* Xh, int64_t ldx, int64_t M, int NP, const __half* Whi,
                   const __half* Wlo, const int* act, int n_coarse, int L_act, int64_t slot_len, int S, float* Gp, int64_t cap,
                   const int* cnt, bool lo_capable, const Upload& up, const SplitOut& so, const int8_t* xshift) {
  if (L_act <= 0) return 0;
#ifdef OICA_EXPERIMENTS
  static bool force_lo = getenv("OICA_TC_FORCE_LO") != nullptr;   // LO-capable layout always
  lo_capable = lo_capable || force_lo;
#endif
  if (lo_capable || n_coarse < L_act)   // fine rows (possibly): LO-capable layout, 2nd pass from tile n_coarse/128
    launch_np<true>(st, Xh, ldx, M, NP, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, n_coarse, cnt, up, so, xshift);
  else
    launch_np<false>(st, Xh, ldx, M, NP, Whi, Wlo, act, L_act, slot_len, S, Gp, cap, 0, cnt, up, so, xshift);
  return 1;
}

int launch_x_prepare_f16(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, int NP, int64_t ldx,
                         __half* Xh, int64_t m_lo, int64_t m_hi) {
  if (m_hi < 0) m_hi = ldx;
  if (m_hi <= m_lo) return 0;
  dim3 grid((unsigned)ceil_div((m_hi - m_lo) / 8, 256), (unsigned)NP);   // ldx, m_lo, m_hi multiples of 8
  k_x_prepare_f16<<<grid, 256, 0, st>>>(X, ld, N, M, ldx, Xh, m_lo, m_hi);
  return 1;
}


}  // namespace oica
