// krp_sketch_tc.cu — the fused all-mode KRP sketch on sm_100a tensor cores (3xTF32).
//
// Method (Alg. 7 line 3 with memoization).  Split the modes into
// rows [0,m), cols [m,m2) and slices [m2,d); X is then an M x C x S array (first index
// fastest, a free reshape).  With W_L(ρ,r) = Π_{k<m} Ω_k(i_k(ρ),r), W_R(γ,r) =
// Π_{m<=k<m2} Ω_k(i_k(γ),r) and Ω_S(s,r) = Π_{k>=m2} Ω_k(i_k(s),r), every Y_n is a
// multi-TTV of one of three small objects:
//     A1(ρ,r) = Σ_s Ω_S(s,r) Σ_γ X(ρ,γ,s) W_R(γ,r)            -> row modes
//     A2(γ,r) = Σ_s Ω_S(s,r) Σ_ρ X(ρ,γ,s) W_L(ρ,r)            -> col modes
//     T(s,r)  = Σ_ρ W_L(ρ,r) Σ_γ X(ρ,γ,s) W_R(γ,r)            -> slice modes
// (all 4·N·R flops, every element of X read from HBM once).  One 128x128 tile X(ρ-block,
// γ-block, s) is loaded by TMA into shared memory; both contractions run on tcgen05:
//     z1 = X_tile · W_R(γ-block)     (M = ρ, K = γ)
//     z2 = X_tileᵀ · W_L(ρ-block)    (M = γ, K = ρ)
// in 3xTF32 (x = hi + lo with hi = x truncated to tf32 — what the tensor core reads, measured
// in tools/tcprobe.cu — and lo = x - hi exact in fp32; products hi·hi + hi·lo + lo·hi, fp32
// accumulation in TMEM).  The Khatri-Rao rows W_R / W_L are formed in registers by the
// epilogue warps once per (ρ-block, γ-block) segment, split into hi/lo and stored in shared
// memory as the UMMA B operand [B_hi | B_lo] (N = 2R, one MMA gives hi·hi and hi·lo); they
// are never materialised in global memory.  A (the tile) is staged by 4 "split" warps into
// TMEM, in both orientations (lane = ρ for z1, lane = γ for z2), as hi and lo.
// The epilogue drains z1/z2 per tile: A1 += z1·Ω_S and A2 += z2·Ω_S in registers, and
// T(s) = Σ_lanes z1·W_L by a warp-shuffle transposed reduction + a fixed-order cross-warp sum.
// A second kernel (fixed order) sums the per-CTA partials and applies the multi-TTVs.
//
// Warp roles (704 threads): 0-3 split (TMEM lane quarters 0-3), 4-19 epilogue ((P|Q side) x
// (r-half) x lane quarter), 20 TMA producer, 21 MMA issuer.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "krp_common.cuh"
#include "krp_internal.h"
#include "sm100.cuh"

namespace krp {
namespace {
using namespace sm100;

// Five warpgroups.  setmaxnreg moves registers from the producer group to the epilogue groups.
constexpr int kNumSplitWarps = 8;  // WG0-1: two per TMEM lane quarter; warp w fills chunk slot w / 4
constexpr int kEpiWarp0 = 8;       // WG2-3: (P | Q side) x TMEM lane quarter
constexpr int kNumEpiWarps = 8;
constexpr int kTmaWarp = 16;       // WG4: TMA producer, MMA issuer (owns the TMEM allocation), 2 idle warps
constexpr int kMmaWarp = 17;
constexpr int kOmsWarp = 18;       // forms each tile's slice Khatri-Rao row Ω_S(s, ·) into a shared-memory ring
constexpr int kOmsSlots = 4;
constexpr int kThreads = 20 * 32;
#ifndef KRP_REGS_PROD
#define KRP_REGS_PROD 32
#endif
#ifndef KRP_REGS_EPI
#define KRP_REGS_EPI 128
#endif
constexpr int kRegsSplit = 96, kRegsEpi = KRP_REGS_EPI, kRegsProd = KRP_REGS_PROD;
// With the A1/A2 accumulators in TMEM or few of them in registers (RA <= 32) the epilogue fits in 112
// registers and the TMA / MMA warps get 48 (at 32 the MMA issue loop spills: 65 local loads / stores in
// <16, 0>, the c5 plan); wider register accumulators keep 128 / 32.  Budget: 256 x (epi - 96) <=
// 128 x (96 - prod).
constexpr int regs_prod(int ra) { return ra <= 32 ? 48 : kRegsProd; }
constexpr int regs_epi(int ra) { return ra <= 32 ? 112 : kRegsEpi; }  // the epilogue gains exactly what the producer group releases: 256*(128-96) = 128*(96-32)
// QH plans (Q's A_hi staged in TMEM, register accumulators up to R8 = 64): the split warps give up 32
// registers too, so the epilogue holds A1 / A2 (64 floats) and the W rows: 256*(152-96) = 256*(96-64) +
// 128*(96-48).
constexpr int kRegsSplitQH = 64, kRegsProdQH = 48, kRegsEpiQH = 152;
constexpr int kTile = 128;
constexpr int kStageFloats = 4 * 128 * 32;  // one 128x128 fp32 tile = 4 TMA boxes of {32, 128}
constexpr int kMaxTcR = 64;

struct TcParams {
  int64_t M, C, S;
  int RB, CB;
  int64_t T;
  int R, NP, N2, R8;  // NP: B-image rows; R8 = round8(R): row of B_lo / column of the hi·lo accumulator
  int triple;         // 1: three N=N2 MMAs into one accumulator (hh + hl + lh); 0: [hi|lo] concat (N=NP) + lo·hi
  int DN;             // accumulator columns per side (NP for concat, N2 for triple)
  int NS, NC, NA;
  int do_p, do_q, do_t;
  int maxseg;  // max number of CTAs contributing to one (rb, cb) pair: partial slot = pair*maxseg + k
  int tm_acc, tm_chunk, tm_a;  // TMEM columns: accumulator stages, A-operand chunk stages, A1/A2
  uint32_t sm_x, sm_bp, sm_bq, sm_red, sm_bar, sm_ws;
  float* partA1;  // [npairs*maxseg][R][128]
  float* partA2;
  int* slot_pair;  // [nslot]
  float* Tpart;    // [RB*CB][S][R]
  // the Ω_k (inputs, I_k x ldo row-major; null: a mode whose Ω is not given, factor 1) and the mode
  // geometry: mode k of a group has index (lin / gs[k]) % n[k].  The Khatri-Rao rows W_L, W_R, Ω_S are
  // formed from these on chip; no table of them exists in global memory.
  const float* om[kMaxD];
  uint32_t gn[kMaxD], ggs[kMaxD];
  int d, m, m2, ldo;
  long long* trace;    // development timeline (KRP_TC_TRACE): CTA 0 role timestamps, null in production
  uint32_t wait_ns;    // mbarrier try_wait suspend-time hint (ns); 0 = spin
  int mma_spin;        // 1: the MMA warp polls its barriers without a suspend hint
  int split_spin;      // 1: the split warps poll chunk_ready without a suspend hint
  int dbg;             // development probes (KRP_TC_DEBUG bits): 1 no TMA data movement, 2 no MMAs, 4 no
                       // epilogue math; results are garbage when set.  Legacy description follows:
                       // 2 TMA + split, 3 TMA + split + MMA (no epilogue), 4 TMA self-consumed
};

// floor(num / den) for 0 <= num < 2^62, den > 0, without the 64-bit integer division routine
__host__ __device__ __forceinline__ int64_t fdiv64(int64_t num, int64_t den) {
  int64_t q = static_cast<int64_t>(static_cast<double>(num) / static_cast<double>(den));
  while (q * den > num) --q;
  while ((q + 1) * den <= num) ++q;
  return q;
}
// CTA owning tile t under the static split a0(b) = floor(b*T/grid): the largest b with a0(b) <= t
__host__ __device__ __forceinline__ int cta_of_tile(int64_t t, int64_t T, int grid) {
  return static_cast<int>(fdiv64((t + 1) * grid - 1, T));
}

// every other wait of the sketch kernel: try_wait with a 10 ms suspend-time hint (development builds:
// the hint / nanosleep back-off / plain spin is chosen by KRP_TC_WAIT_NS)
#ifdef KRP_DEV_TRACE
#define KWAIT(bar, par)                                              \
  do {                                                               \
    if (p.wait_ns >= 100000) mbar_wait_hint((bar), (par), p.wait_ns); \
    else if (p.wait_ns) mbar_wait_sleep((bar), (par), p.wait_ns);    \
    else mbar_wait_spin((bar), (par));                               \
  } while (0)
#else
#define KWAIT(bar, par) mbar_wait_hint((bar), (par), 10000000u)
#endif

// Development timeline (CTA 0 role timestamps): compiled in only with -DKRP_DEV_TRACE, so the
// production kernel carries no per-chunk trace checks.
#ifdef KRP_DEV_TRACE
#define KRP_TRACE(slot, idx)                                                                 \
  do {                                                                                       \
    if (p.trace && blockIdx.x == 0 && (idx) < 64) p.trace[(slot) * 64 + (idx)] = clock64(); \
  } while (0)
#else
#define KRP_TRACE(slot, idx) \
  do {                       \
  } while (0)
#endif
// Development probes (TcParams::dbg bits: disable TMA data / MMAs / epilogue math ...) and the
// wait-mode switches exist only in KRP_DEV_TRACE builds; production always spins on the hot barriers.
#ifdef KRP_DEV_TRACE
#define KRP_DBG(bit) ((p.dbg & (bit)) != 0)
#define KRP_MMA_SPIN (p.mma_spin != 0)
#define KRP_SPLIT_SPIN (p.split_spin != 0)
#elif defined(KRP_PROBE_BITS)  // development: compile-time probes in an otherwise production build
#define KRP_DBG(bit) ((KRP_PROBE_BITS & (bit)) != 0)
#define KRP_MMA_SPIN true
#define KRP_SPLIT_SPIN true
#else
#define KRP_DBG(bit) false
#define KRP_MMA_SPIN true
#define KRP_SPLIT_SPIN true
#endif
// hot-barrier polling: 0 = spin on try_wait; > 0 = nanosleep back-off of that many ns between probes
// (a sleeping warp leaves its SMSP's issue slots to the split / epilogue warps sharing it)
// Measured (profiles/r01j_ab_mma_backoff.log): a 32 ns back-off of the MMA warp's polls helps the wide
// register-accumulator plans (R8 >= 32: c2 -1.5 %, c3 -1.2 %) and hurts the narrow ones (c4 +3 %), so by
// default it is applied per instantiation (RA >= 32).
// Split-warp roles (profiles/r01j_ab_split_roles.log): with roles, the two warps of a lane quarter share
// every chunk (P hi / P lo vs Q lo); without, each takes alternate chunks.  Both warps issue from the
// same SMSP, so roles only pay where the TMEM-accumulator plan leaves the split latency exposed
// (RA == 0: c5 -3 %); elsewhere alternate chunks are faster (c4 +3..13 % with roles).  -1 = per plan.
#ifndef KRP_SPLIT_ROLES
#define KRP_SPLIT_ROLES -1
#endif
#ifndef KRP_MMA_SLEEP_NS
#define KRP_MMA_SLEEP_NS (RA >= 32 ? 32 : 0)
#endif
#ifndef KRP_BUILD_BATCH
#define KRP_BUILD_BATCH 8
#endif
#ifndef KRP_SKETCH_PDL
#define KRP_SKETCH_PDL 0
#endif
// L2 prefetch distance of the TMA producer, in tiles; -1 = per plan (profiles/r02o_ab_prefetch_distance.log:
// with >= 2 shared-memory stages the TMA loads themselves run far enough ahead and the extra prefetch requests
// cost 2 % at c2-c4; with c5's single stage one tile ahead pays, deeper distances lose everywhere)
#ifndef KRP_PF
#define KRP_PF -1
#endif
#ifndef KRP_SPLIT_BATCH
#define KRP_SPLIT_BATCH 1
#endif
#ifndef KRP_SPLIT_SLEEP_NS
#define KRP_SPLIT_SLEEP_NS 0
#endif
#define HOT_WAIT(bar, par, ns)                                  \
  do {                                                          \
    if ((ns) > 0) mbar_wait_sleep((bar), (par), (ns) > 0 ? (ns) : 1); \
    else mbar_wait_spin((bar), (par));                          \
  } while (0)

__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

__device__ __forceinline__ float lds_f32(uint32_t saddr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t saddr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(saddr), "f"(v) : "memory");
}

// One 8-column epilogue round for this thread's TMEM lane: z = D[rr..rr+8) (+ D[R8+rr..] for the concat
// form), acc += z·Ω_S; on this side's T rounds, the 32-lane transposed butterfly of z·W is written to rbuf.
// w holds this lane's Khatri-Rao row W(lane, rr..rr+8) (registers, loaded once per segment); the Ω_S row of
// the tile is read with two 16-byte loads (rows are R8 floats, zero padded).  Adds / fmas run two-wide.
// The two halves of a round: drain (TMEM -> z, masked) and math (acc += z·Ω_S; T butterfly).
__device__ __forceinline__ void epi_drain8(int rnd, float (&z)[8], uint32_t tD, int R, int R8, int triple) {
  const int rr = 8 * rnd;
  float a[8], b[8];
  tmem_ld8(tD + rr, a);
  if (!triple) tmem_ld8(tD + R8 + rr, b);
  tmem_ld_wait();
  const bool full = rr + 8 <= R;
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    float2 v = make_float2(a[j], a[j + 1]);
    if (!triple) v = f2_add(v, make_float2(b[j], b[j + 1]));
    if (!full) {  // columns >= R of the accumulator hold padding (possibly stale TMEM): zero them
      v.x = rr + j < R ? v.x : 0.f;
      v.y = rr + j + 1 < R ? v.y : 0.f;
    }
    z[j] = v.x;
    z[j + 1] = v.y;
  }
}
__device__ __forceinline__ void epi_math8(int rnd, const float (&z)[8], float (&acc)[8], uint32_t oms_s,
                                          bool my_t, const float (&w)[8], uint32_t rbuf_s, int R8, uint32_t sub,
                                          uint32_t lane) {
  const int rr = 8 * rnd;
  float om[8], tv[8];
  // Ω_S(s, rr..rr+8): the tile's slice Khatri-Rao row, formed by the MMA warp in shared memory (zero padded)
  lds_v4(oms_s + rr * 4, om[0], om[1], om[2], om[3]);
  lds_v4(oms_s + rr * 4 + 16, om[4], om[5], om[6], om[7]);
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float2 zz = make_float2(z[j], z[j + 1]);
    const float2 c = f2_fma(zz, make_float2(om[j], om[j + 1]), make_float2(acc[j], acc[j + 1]));
    acc[j] = c.x;
    acc[j + 1] = c.y;
    if (my_t) {
      const float2 t = f2_mul(zz, make_float2(w[j], w[j + 1]));
      tv[j] = t.x;
      tv[j + 1] = t.y;
    }
  }
  if (my_t) {
#pragma unroll
    for (int lvl = 0; lvl < 3; ++lvl) {
      const int m = 16 >> lvl;
      const int h = 4 >> lvl;
      const bool upper = (lane & m) != 0;
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float send = upper ? tv[j] : tv[j + h];
        const float keep = upper ? tv[j + h] : tv[j];
        tv[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    }
    tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 2);
    tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 1);
    if ((lane & 3) == 0) sts_f32(rbuf_s + (sub * R8 + rr + (lane >> 2)) * 4, tv[0]);
  }
}

__device__ __forceinline__ void epi_round8(int rnd, float (&acc)[8], uint32_t tD, int R, int R8, int triple,
                                           uint32_t oms_s, bool my_t, const float (&w)[8], uint32_t rbuf_s,
                                           uint32_t sub, uint32_t lane) {
  const int rr = 8 * rnd;
  float a[8], b[8], om[8], tv[8];
  tmem_ld8(tD + rr, a);
  if (!triple) tmem_ld8(tD + R8 + rr, b);
  lds_v4(oms_s + rr * 4, om[0], om[1], om[2], om[3]);  // Ω_S(s, rr..rr+8) (shared memory, zero padded)
  lds_v4(oms_s + rr * 4 + 16, om[4], om[5], om[6], om[7]);
  tmem_ld_wait();
  const bool full = rr + 8 <= R;
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    float2 z = make_float2(a[j], a[j + 1]);
    if (!triple) z = f2_add(z, make_float2(b[j], b[j + 1]));
    if (!full) {  // columns >= R of the accumulator hold padding (possibly stale TMEM): zero them
      z.x = rr + j < R ? z.x : 0.f;
      z.y = rr + j + 1 < R ? z.y : 0.f;
    }
    const float2 c = f2_fma(z, make_float2(om[j], om[j + 1]), make_float2(acc[j], acc[j + 1]));
    acc[j] = c.x;
    acc[j + 1] = c.y;
    if (my_t) {
      const float2 t = f2_mul(z, make_float2(w[j], w[j + 1]));
      tv[j] = t.x;
      tv[j + 1] = t.y;
    }
  }
  if (my_t) {
    // 3 halving levels + 2 plain levels: lanes 4q..4q+3 end with the 32-lane sum for r = rr + q
#pragma unroll
    for (int lvl = 0; lvl < 3; ++lvl) {
      const int m = 16 >> lvl;
      const int h = 4 >> lvl;
      const bool upper = (lane & m) != 0;
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float send = upper ? tv[j] : tv[j + h];
        const float keep = upper ? tv[j + h] : tv[j];
        tv[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    }
    tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 2);
    tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 1);
    if ((lane & 3) == 0) sts_f32(rbuf_s + (sub * R8 + rr + (lane >> 2)) * 4, tv[0]);
  }
}

// CH: TMEM A-operand chunk width (K columns per split/MMA handshake); RA: 0 = A1/A2 accumulators in
// TMEM, else they live in registers (RA = R8, a multiple of 8).
//
// Synchronisation (all mbarriers; g = the CTA's running chunk index, cst = g % NC):
//   full_x[st]      TMA landed tile stage st                          (producer tx; split + MMA warps wait)
//   empty_x[st]     stage st may be overwritten                       (4 split arrivals + 1 MMA commit)
//   chunk_ready[c]  chunk slot c is free: its previous MMAs are done  (1 MMA commit; split waits)
//   chunk_full[c]   split wrote P hi / P lo / Q lo of the chunk       (4 split arrivals; MMA waits)
//   acc_full[a]     the tile's accumulators are complete              (1 MMA commit; epilogue waits)
//   oms_full[o]     the tile's Ω_S row is in ring slot o              (32 Ω_S-warp lanes; epilogue waits)
//   oms_empty[o]    the epilogue is done with ring slot o             (8 epilogue warps; Ω_S warp waits)
//   acc_empty[a]    the epilogue drained accumulator stage a          (8 epilogue arrivals; MMA waits)
//   b_ready         the segment's B images are in shared memory      (1 epilogue arrival; MMA waits)
//
// QH (Q's A_hi in TMEM): the split warps also store the raw tile with lane = γ, so no MMA reads the tile
// stage; it is released as soon as the split warps have read it (they run up to NC chunks ahead of the
// MMA), and the next tile's TMA overlaps the MMAs of the current one even with a single stage (NS = 1).
template <int CH, int RA, bool QH = false>
__global__ void __launch_bounds__(kThreads, 1)
    krp_tc_sketch_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TcParams p) {
  constexpr bool kSplitRoles = KRP_SPLIT_ROLES < 0 ? (RA == 0 || QH) : (KRP_SPLIT_ROLES != 0);
  constexpr int kSlot = (QH ? 4 : 3) * CH;  // TMEM columns of one chunk slot: [P hi | P lo | Q lo (| Q hi)]
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xs = reinterpret_cast<float*>(smem + p.sm_x);
  uint8_t* bp = smem + p.sm_bp;
  uint8_t* bq = smem + p.sm_bq;
  float* red = reinterpret_cast<float*>(smem + p.sm_red);  // [2 parities][4 lane quarters][R8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.sm_bar);
  uint64_t* full_x = bars;
  uint64_t* empty_x = full_x + p.NS;
  uint64_t* chunk_full = empty_x + p.NS;
  uint64_t* chunk_ready = chunk_full + p.NC;
  uint64_t* acc_full = chunk_ready + p.NC;
  uint64_t* acc_empty = acc_full + p.NA;
  uint64_t* b_ready = acc_empty + p.NA;
  uint64_t* oms_full = b_ready + 1;
  uint64_t* oms_empty = oms_full + kOmsSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(oms_empty + kOmsSlots);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (threadIdx.x == 0) KRP_TRACE(13, 56);  // (development timeline: kernel entry)
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&full_x[i], 1);
      mbar_init(&empty_x[i], QH ? kNumSplitWarps : kNumSplitWarps + 1);  // split warps (+ the MMA warp's commit)
    }
    for (int i = 0; i < p.NC; ++i) {
      mbar_init(&chunk_full[i], kSplitRoles ? kNumSplitWarps : 4);  // split warps writing this slot
      mbar_init(&chunk_ready[i], 1);
    }
    for (int i = 0; i < p.NA; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kNumEpiWarps);
    }
    mbar_init(b_ready, 1);
    for (int i = 0; i < kOmsSlots; ++i) {
      mbar_init(&oms_full[i], 32);
      mbar_init(&oms_empty[i], kNumEpiWarps);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (threadIdx.x == 0) KRP_TRACE(13, 57);  // prologue done
  pdl_launch_dependents();  // the assembly kernel may be scheduled now (it waits for this grid to finish)
#if KRP_SKETCH_PDL
  pdl_wait();  // launched as a programmatic dependent: X and the Ω_k are read only after the previous grid
#endif

  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * p.T / gridDim.x;
  const int64_t t1 = static_cast<int64_t>(blockIdx.x + 1) * p.T / gridDim.x;
  constexpr int nkc = kTile / CH;
  const int64_t nchunks = (t1 - t0) * nkc;

  if (warp >= kTmaWarp) {
  // producer warpgroup: one setmaxnreg for the whole group, then TMA / MMA / idle warps
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(QH ? kRegsProdQH : regs_prod(RA)));
  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmap);
      const uint64_t pol = policy_evict_first();
      int st = 0;
      uint32_t ph = 0;
      int64_t pair = t0 / p.S, s = t0 % p.S;
      int rb = static_cast<int>(pair / p.CB), cb = static_cast<int>(pair % p.CB);
      // L2 prefetch runs kPf tiles ahead of the loads: only where a single SMEM stage leaves the loads no lead
      const int kPf = KRP_PF >= 0 ? KRP_PF : (p.NS >= 2 ? 0 : 1);
      int64_t pf_t = t0, pf_pair = pair, pf_s = s;
      auto pf_issue = [&]() {
        const int pp = static_cast<int>(pf_pair), prb = pp / p.CB, pcb = pp - prb * p.CB;  // 32-bit division
        for (int j = 0; j < 4; ++j) tma_prefetch_3d(&tmap, prb * kTile + 32 * j, pcb * kTile, static_cast<int32_t>(pf_s));
        if (++pf_s == p.S) {
          pf_s = 0;
          ++pf_pair;
        }
        ++pf_t;
      };
      for (int i = 0; i < kPf && pf_t < t1; ++i) pf_issue();
      for (int64_t t = t0; t < t1; ++t) {
        if (kPf > 0 && pf_t < t1) pf_issue();
        KWAIT(&empty_x[st], ph ^ 1);
        KRP_TRACE(0, t - t0);
        if (KRP_DBG(1)) {  // probe: no data movement (the stage holds whatever it held)
          mbar_arrive(&full_x[st]);
        } else {
          mbar_arrive_expect_tx(&full_x[st], kStageFloats * 4);
          float* dst = xs + st * kStageFloats;
          for (int j = 0; j < 4; ++j)
            tma_load_3d(dst + j * 4096, &tmap, &full_x[st], rb * kTile + 32 * j, cb * kTile, static_cast<int32_t>(s),
                        pol);
        }
        if (++st == p.NS) {
          st = 0;
          ph ^= 1;
        }
        if (++s == p.S) {
          s = 0;
          ++pair;
          rb = static_cast<int>(pair / p.CB);
          cb = static_cast<int>(pair % p.CB);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (both GEMMs)
    // The whole warp runs the loop (warp-uniform descriptors in uniform registers); one elected lane
    // issues.  Descriptors advance by (byte offset >> 4) on the start-address field.
    const bool leader = elect_one();
    const uint32_t idesc1 = make_idesc_tf32(128, p.NP, 0, 0);
    const uint32_t idesc2 = make_idesc_tf32(128, p.N2, 0, 0);
    const uint64_t bpdesc0 = make_smem_desc(smem_u32(bp), 0, 1024, kLayoutSW128);
    const uint64_t bqdesc0 = make_smem_desc(smem_u32(bq), 0, 1024, kLayoutSW128);
    const uint64_t adesc0 = make_smem_desc(smem_u32(xs), 0, 1024, kLayoutSW128);
    const uint64_t lo_d = static_cast<uint64_t>(p.R8) * 8;     // B_lo rows start at R8: (R8*128 B) >> 4
    const uint64_t katom_d = static_cast<uint64_t>(p.NP) * 8;  // one 32-wide K atom of B: (NP*128 B) >> 4
    int ast = 0, xst = 0, cst = 0;
    uint32_t aph = 0, bph = 0, cph = 0;
    int64_t s_cur = t0 % p.S;
    bool first = true;
    for (int64_t t = t0; t < t1; ++t) {
      if (first || s_cur == 0) {  // a new (row block, col block) segment: wait for its B operands
        KWAIT(b_ready, bph);
        bph ^= 1;
        first = false;
      }
      if (KRP_MMA_SPIN) HOT_WAIT(&acc_empty[ast], aph ^ 1, KRP_MMA_SLEEP_NS); else KWAIT(&acc_empty[ast], aph ^ 1);
      if (leader) KRP_TRACE(3, t - t0);
      tc_fence_after();
      const uint32_t dP = tbase + p.tm_acc + ast * 2 * p.DN;
      const uint32_t dQ = dP + p.DN;
        const uint64_t adesc_t = adesc0 + ((static_cast<uint64_t>(xst) * (kStageFloats * 4)) >> 4);
      for (int kc = 0; kc < nkc; ++kc) {
        if (KRP_MMA_SPIN) HOT_WAIT(&chunk_full[cst], cph, KRP_MMA_SLEEP_NS); else KWAIT(&chunk_full[cst], cph);
        if (leader) KRP_TRACE(10, (t - t0) * 8 + kc);
        tc_fence_after();
        const uint32_t ach = tbase + p.tm_chunk + cst * kSlot;  // [P hi | P lo | Q lo (| Q hi)]
        const int kk0 = kc * (CH / 8);
        const uint64_t boff = static_cast<uint64_t>(kk0 >> 2) * katom_d + (kk0 & 3) * 2;
        // Q's A_hi: the raw tile in stage xst, box kk0/4 (16 KB), K offset (kk0 & 3) * 32 B
        const uint64_t aq = adesc_t + static_cast<uint64_t>(kk0 >> 2) * 1024 + (kk0 & 3) * 2;
        if (leader && !KRP_DBG(2)) {  // probe bit 2: no MMAs (handshakes only)
          if (p.triple) {
#pragma unroll
            for (int ks = 0; ks < CH / 8; ++ks) {
              const uint32_t acc0 = (kk0 + ks) > 0 ? 1u : 0u;
              const uint64_t bd = bpdesc0 + boff + ks * 2, bdq = bqdesc0 + boff + ks * 2;
              mma_tf32_ts(dP, ach + 8 * ks, bd, idesc2, acc0);              // P: hi x hi
              mma_tf32_ts(dP, ach + 8 * ks, bd + lo_d, idesc2, 1u);         //    hi x lo
              mma_tf32_ts(dP, ach + CH + 8 * ks, bd, idesc2, 1u);           //    lo x hi
              if constexpr (QH) {
                mma_tf32_ts(dQ, ach + 3 * CH + 8 * ks, bdq, idesc2, acc0);  // Q: hi (TMEM) x hi
                mma_tf32_ts(dQ, ach + 3 * CH + 8 * ks, bdq + lo_d, idesc2, 1u);  //  hi x lo
              } else {
                mma_tf32_ss(dQ, aq + ks * 2, bdq, idesc2, acc0);            // Q: hi (SMEM) x hi
                mma_tf32_ss(dQ, aq + ks * 2, bdq + lo_d, idesc2, 1u);       //    hi x lo
              }
              mma_tf32_ts(dQ, ach + 2 * CH + 8 * ks, bdq, idesc2, 1u);      //    lo x hi
            }
          } else {
#pragma unroll
            for (int ks = 0; ks < CH / 8; ++ks) {
              const uint32_t acc0 = (kk0 + ks) > 0 ? 1u : 0u;
              const uint64_t bd = bpdesc0 + boff + ks * 2, bdq = bqdesc0 + boff + ks * 2;
              mma_tf32_ts(dP, ach + 8 * ks, bd, idesc1, acc0);              // P: hi x [B_hi | B_lo]
              mma_tf32_ts(dP, ach + CH + 8 * ks, bd, idesc2, 1u);           //    lo x B_hi
              mma_tf32_ss(dQ, aq + ks * 2, bdq, idesc1, acc0);              // Q: hi (SMEM) x [B_hi | B_lo]
              mma_tf32_ts(dQ, ach + 2 * CH + 8 * ks, bdq, idesc2, 1u);      //    lo x B_hi
            }
          }
        }
        if (leader) {
          mma_commit(&chunk_ready[cst]);  // the slot is free again once these MMAs finish
          KRP_TRACE(11, (t - t0) * 8 + kc);
        }
        __syncwarp();
        if (++cst == p.NC) {
          cst = 0;
          cph ^= 1;
        }
      }
      if (leader) {
        if constexpr (!QH) mma_commit(&empty_x[xst]);  // the raw tile (Q's A_hi) may be overwritten once these MMAs finish
        mma_commit(&acc_full[ast]);
        KRP_TRACE(4, t - t0);
      }
      __syncwarp();
      if (++xst == p.NS) xst = 0;
      if (++ast == p.NA) {
        ast = 0;
        aph ^= 1;
      }
      if (++s_cur == p.S) s_cur = 0;
    }
  } else if (warp == kOmsWarp) {
    // ------------------------------------------------------------ Ω_S warp (otherwise idle)
    // Ω_S(s, r) = Π_{k>=m2} Ω_k(i_k(s), r), lane r and r + 32, for each tile in order into ring slot
    // (t - t0) % kOmsSlots: runs up to kOmsSlots tiles ahead of the epilogue, so the Ω loads' latency is
    // off every other role's path.  The row is formed from the Ω_k inputs (never tabulated in HBM).
    float* ring = reinterpret_cast<float*>(smem + p.sm_ws);
    int o = 0;
    uint32_t oph = 0;
    uint32_t sl = static_cast<uint32_t>(t0 % p.S);
    for (int64_t t = t0; t < t1 && !KRP_DBG(512); ++t) {
      KWAIT(&oms_empty[o], oph ^ 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = static_cast<int>(lane) + 32 * h;
        float w = r < p.R ? 1.f : 0.f;
        if (r < p.R)
          for (int k = p.m2; k < p.d; ++k)
            if (p.om[k]) w *= __ldg(p.om[k] + static_cast<size_t>((sl / p.ggs[k]) % p.gn[k]) * p.ldo + r);
        ring[o * kMaxTcR + r] = w;
      }
      mbar_arrive(&oms_full[o]);  // release: this lane's row entries
      if (++o == kOmsSlots) {
        o = 0;
        oph ^= 1;
      }
      if (++sl == static_cast<uint32_t>(p.S)) sl = 0;
    }
  }
  } else if (warp < kNumSplitWarps) {
    // (two split warps per lane quarter: warp w processes the chunks of slot w / 4, i.e. kc % 2 == w / 4)
    // ------------------------------------------------------------ split warps: tile -> TMEM hi / lo
    // P view (lane = ρ): shared-memory loads (the transpose), hi = raw value, lo = x - tf32(x).
    // Q view (lane = γ): 16-byte loads of the rows; only lo goes to TMEM (Q's hi is read from SMEM).
    if constexpr (QH) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsSplitQH));
    const uint32_t sub = warp & 3;
    // kSplitRoles: the two warps of a lane quarter share every chunk, warp w < 4 writing P hi / P lo and
    // warp w >= 4 Q lo (halves the split latency of a chunk); else warp w takes the chunks kc % 2 == w / 4.
    const int par = static_cast<int>(warp >> 2);
    const uint32_t lane_off = (32u * sub) << 16;
    int xst = 0;
    uint32_t xph = 0;
    const bool dop = p.do_p != 0 && (!kSplitRoles || par == 0), doq = p.do_q != 0 && (!kSplitRoles || par == 1);
    // P view: element (ρ = 32*sub + lane, γ) of box `sub` sits at byte γ*128 + (((lane>>2) ^ (γ&7)) << 4) +
    // (lane&3)*4; γ&7 is the compile-time j&7 below, so every load is register + immediate.
    uint32_t psw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      psw[j] = smem_u32(xs) + sub * 16384u + ((((lane >> 2) ^ static_cast<uint32_t>(j)) << 4) | ((lane & 3u) << 2));
    const uint32_t gq = 32 * sub + lane;
    const uint32_t qrow = smem_u32(xs) + gq * 128u, qx = gq & 7u;
    // chunk g of the CTA (all tiles) sits in slot g % NC; this warp takes the chunks with g % 2 == par
    // (nkc is even, so that is kc % 2 == par in every tile); (cst, cph) track slot and phase of chunk g
    int cst = 0;
    uint32_t cph = 0;
    auto advance = [&]() {
      if (++cst == p.NC) {
        cst = 0;
        cph ^= 1;
      }
    };
    if (!kSplitRoles && par) advance();
    constexpr int kcStep = kSplitRoles ? 1 : 2;
    // kBatch chunks per wait::st / fence / arrive round (roles mode): amortises the per-chunk handshake
    constexpr int kBatch = kSplitRoles ? KRP_SPLIT_BATCH : 1;
    for (int64_t t = t0; t < t1; ++t) {
      KWAIT(&full_x[xst], xph);
      if (sub == 0 && lane == 0) KRP_TRACE(1, t - t0);
      const uint32_t stage_off = static_cast<uint32_t>(xst) * (kStageFloats * 4u);
      for (int kc0 = kSplitRoles ? 0 : par; kc0 < nkc; kc0 += kcStep * kBatch) {
        if (sub == 0 && lane == 0) KRP_TRACE(13, (t - t0) * 8 + kc0);
        int bst[kBatch];
        {
          int c = cst;
          uint32_t ph = cph;
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            bst[b] = c;
            if (KRP_SPLIT_SPIN) HOT_WAIT(&chunk_ready[c], ph ^ 1, KRP_SPLIT_SLEEP_NS); else KWAIT(&chunk_ready[c], ph ^ 1);
            if (++c == p.NC) {
              c = 0;
              ph ^= 1;
            }
          }
        }
        if (sub == 0 && lane == 0) KRP_TRACE(8, (t - t0) * 8 + kc0);
        tc_fence_after();
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
        const int kc = kc0 + b;
        const uint32_t ch = tbase + lane_off + p.tm_chunk + bst[b] * kSlot;
        // P view: CH scalar loads (lane = ρ), hi stored as loaded, lo formed in place and stored
        if (dop && !KRP_DBG(8) && !KRP_DBG(128)) {  // probe bits 8: no split work, 128: no P-view split
          uint32_t px[CH];
          const uint32_t goff = stage_off + static_cast<uint32_t>(kc * CH) * 128u;
#pragma unroll
          for (int j = 0; j < CH; ++j) px[j] = __float_as_uint(lds_f32(psw[j & 7] + goff + static_cast<uint32_t>(j) * 128u));
          if (sub == 0 && lane == 0) KRP_TRACE(14, (t - t0) * 8 + kc);
          tmem_st<CH>(ch + 0 * CH, px);  // hi: the raw value (the tensor core truncates to tf32)
#pragma unroll
          for (int j = 0; j < CH; j += 2) {
            const float2 x = make_float2(__uint_as_float(px[j]), __uint_as_float(px[j + 1]));
            const float2 l = f2_sub(x, make_float2(__uint_as_float(tf32_hi_bits(x.x)), __uint_as_float(tf32_hi_bits(x.y))));
            px[j] = __float_as_uint(l.x);
            px[j + 1] = __float_as_uint(l.y);
          }
          tmem_st<CH>(ch + 1 * CH, px);
        }
        // Q view: lane = γ, columns ρ = kc*CH + j: CH consecutive ρ of row γ (16-byte chunks, swizzled)
        if (doq && !KRP_DBG(8)) {
          uint32_t qv[CH];
          const int rho0 = kc * CH;
          const uint32_t rowa = qrow + stage_off + static_cast<uint32_t>(rho0 >> 5) * 16384u;
#pragma unroll
          for (int qq = 0; qq < CH / 4; ++qq) {
            const uint32_t chunk = ((static_cast<uint32_t>(rho0 & 31) >> 2) + qq) ^ qx;
            float a0, a1, a2, a3;
            lds_v4(rowa + (chunk << 4), a0, a1, a2, a3);
            qv[4 * qq] = __float_as_uint(a0), qv[4 * qq + 1] = __float_as_uint(a1);
            qv[4 * qq + 2] = __float_as_uint(a2), qv[4 * qq + 3] = __float_as_uint(a3);
          }
          if constexpr (QH) tmem_st<CH>(ch + 3 * CH, qv);  // Q hi: the raw value
#pragma unroll
          for (int j = 0; j < CH; j += 2) {
            const float2 x = make_float2(__uint_as_float(qv[j]), __uint_as_float(qv[j + 1]));
            const float2 l = f2_sub(x, make_float2(__uint_as_float(tf32_hi_bits(x.x)), __uint_as_float(tf32_hi_bits(x.y))));
            qv[j] = __float_as_uint(l.x);
            qv[j + 1] = __float_as_uint(l.y);
          }
          tmem_st<CH>(ch + 2 * CH, qv);  // Q lo
        }
        }  // batch
        if (sub == 0 && lane == 0) KRP_TRACE(15, (t - t0) * 8 + kc0);
        tmem_st_wait();
        if (sub == 0 && lane == 0) KRP_TRACE(9, (t - t0) * 8 + kc0);
        tc_fence_before();
        __syncwarp();
        if (sub == 0 && lane == 0) KRP_TRACE(12, (t - t0) * 8 + kc0);
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
          if (lane == 0) mbar_arrive(&chunk_full[cst]);
          advance();
          if (!kSplitRoles) advance();  // skip the other parity's chunk
        }
      }
      __syncwarp();
      if (sub == 0 && lane == 0) KRP_TRACE(2, t - t0);
      if (lane == 0) mbar_arrive(&empty_x[xst]);
      if (++xst == p.NS) {
        xst = 0;
        xph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    // warps 8-11: P side (z1 -> A1 += z1·Ω_S), warps 12-15: Q side (z2 -> A2 += z2·Ω_S); A1/A2 live
    // in TMEM (lane = ρ resp. γ).  T(s,r) = Σ_ρ z1·W_L = Σ_γ z2·W_R: its 8-column rounds alternate
    // between the two sides.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(QH ? kRegsEpiQH : regs_epi(RA)));  // both epilogue WGs

    const uint32_t ew = warp - kEpiWarp0;  // 0..7
    const uint32_t sub = warp & 3;         // TMEM lane quarter
    const bool pside = ew < 4;
    const int l = static_cast<int>(32 * sub + lane);
    const uint32_t lane_off = (32u * sub) << 16;
    const uint32_t k32 = static_cast<uint32_t>(l) & 31u, katom = static_cast<uint32_t>(l) >> 5;
    const uint32_t c0 = k32 >> 2, e0 = (k32 & 3u) * 4u;  // swizzle: byte offset in a row = ((c0 ^ (row & 7)) << 4) + e0
    const bool active = pside ? (p.do_p != 0) : (p.do_q != 0);
    const int R = p.R, R8 = p.R8;
    const int nr = (R + 7) / 8;
    // my side's W (B_Q = W_L rows for the P side, B_P = W_R rows for the Q side) for the T rounds
    // this thread's k-atom of the image: row n's element sits at wb + n*128 + ((c0 ^ (n & 7)) << 4) + e0
    const uint32_t wb = smem_u32((pside ? bq : bp) + katom * (p.NP * 128));
    const uint32_t tA = tbase + lane_off + p.tm_a + (pside ? 0 : R8);  // A1 / A2 columns
    // this lane's W row for this side's T rounds (P side: even rounds, Q side: odd rounds)
    constexpr int kRounds = RA > 0 ? RA / 8 : kMaxTcR / 8;
    constexpr int kTRounds = (kRounds + 1) / 2;
    float wreg[8 * kTRounds];
#pragma unroll
    for (int j = 0; j < 8 * kTRounds; ++j) wreg[j] = 0.f;
    const uint32_t zero8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float Areg[RA > 0 ? RA : 1];
#pragma unroll
    for (int j = 0; j < (RA > 0 ? RA : 1); ++j) Areg[j] = 0.f;
    int ast = 0;
    uint32_t aph = 0;
    int64_t prev_pair = -1;
    int seg = -1;
    int oslot = 0;  // Ω_S ring slot of the current tile and its phase
    uint32_t ooph = 0;
    int parity = 0;
    int64_t pair = t0 / p.S, s = t0 % p.S;  // advanced incrementally (no 64-bit division per tile)
    for (int64_t t = t0; t < t1; ++t, (++s == p.S ? (s = 0, ++pair) : 0)) {
      if (pair != prev_pair) {
        if (prev_pair >= 0)
        {  // flush the finished segment's accumulators into its partial slot
          const int kslot = static_cast<int>(blockIdx.x - cta_of_tile(prev_pair * p.S, p.T, gridDim.x));
          const int64_t slot = prev_pair * p.maxseg + kslot;
          if (threadIdx.x == kEpiWarp0 * 32) p.slot_pair[slot] = static_cast<int>(prev_pair);
          // slot layout [r][128]: for a fixed r the 32 lanes of a warp store 128 contiguous bytes
          float* dst = (pside ? p.partA1 : p.partA2) + slot * kTile * R + l;

          if constexpr (RA > 0) {
#pragma unroll
            for (int j = 0; j < RA; ++j) {
              if (active && j < R) dst[j * kTile] = Areg[j];
              Areg[j] = 0.f;
            }
          } else if (active) {
            for (int rnd = 0; rnd < nr; ++rnd) {
              float v[8];
              tmem_ld8(tA + 8 * rnd, v);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (8 * rnd + j < R) dst[(8 * rnd + j) * kTile] = v[j];
            }
          }
        }

        ++seg;
        prev_pair = pair;
        const int64_t rb = pair / p.CB, cb = pair % p.CB;
        // zero this segment's accumulators (register accumulators are zeroed by the flush)
        if (RA == 0 && active) {
          for (int rnd = 0; rnd < nr; ++rnd) tmem_st8(tA + 8 * rnd, zero8);
          tmem_st_wait();
        }
        // B operands of this segment, formed on chip (P side -> B_Q = W_L rows of row block rb, Q side ->
        // B_P = W_R rows of col block cb): this thread's row lin = 128*blk + l of the group is the product of
        // its modes' Ω rows, accumulated in place in the image's hi rows, then split hi / lo (UMMA K-major
        // SWIZZLE_128B layout [k-atom][NP rows][128 B]; rows [R, R8) and [R8 + R, NP) are zero)
        {
          const uint32_t lin = static_cast<uint32_t>((pside ? rb : cb) * kTile) + static_cast<uint32_t>(l);
          const bool inside = lin < static_cast<uint32_t>(pside ? p.M : p.C);
          const int k0 = pside ? 0 : p.m, k1 = pside ? p.m : p.m2;
          // the group's first two given modes' rows (independent loads in flight), further modes through a
          // generic loop; Ω_n of a single-mode sketch is not given (factor 1)
          const float* rowa = nullptr;
          const float* rowb = nullptr;
          int kx = k1;
          if (inside)
            for (int k = k0; k < k1; ++k) {
              if (!p.om[k]) continue;
              const float* row = p.om[k] + static_cast<size_t>((lin / p.ggs[k]) % p.gn[k]) * p.ldo;
              if (!rowa) {
                rowa = row;
              } else if (!rowb) {
                rowb = row;
              } else {
                kx = k;
                break;
              }
            }
          const uint32_t lo_row = static_cast<uint32_t>(R8) * 128u;
          for (int r0 = 0; r0 < R8; r0 += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const bool ok = r0 + j < R;
              const float a = ok && rowa ? __ldg(rowa + r0 + j) : 1.f;
              const float b = ok && rowb ? __ldg(rowb + r0 + j) : 1.f;
              v[j] = ok && inside ? a * b : 0.f;
            }
            for (int k = kx; k < k1; ++k) {
              if (!p.om[k]) continue;
              const float* row = p.om[k] + static_cast<size_t>((lin / p.ggs[k]) % p.gn[k]) * p.ldo;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (r0 + j < R) v[j] *= __ldg(row + r0 + j);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // rows r0 + j: (r0 + j) & 7 == j
              const uint32_t ad = wb + ((c0 ^ static_cast<uint32_t>(j)) << 4) + e0 + static_cast<uint32_t>(r0 + j) * 128u;
              const float whi = __uint_as_float(tf32_hi_bits(v[j]));
              sts_f32(ad, whi);  // rows [R, R8): zero
              if (r0 + j < R) sts_f32(ad + lo_row, v[j] - whi);
            }
          }
          for (int r = R8 + R; r < p.NP; ++r)
            sts_f32(wb + ((c0 ^ static_cast<uint32_t>(r & 7)) << 4) + e0 + static_cast<uint32_t>(r) * 128u, 0.f);
        }
        fence_proxy_async_smem();
        named_bar_sync(1, kNumEpiWarps * 32);
        if (threadIdx.x == kEpiWarp0 * 32) mbar_arrive(b_ready);
        if (threadIdx.x == kEpiWarp0 * 32 && seg == 0) KRP_TRACE(13, 59);  // first B images ready
        if (p.do_t) {  // W(lane, r) = hi + lo rows of the image just copied (B_Q for the P side, B_P for Q)
          const uint32_t lo_row = static_cast<uint32_t>(R8) * 128;
#pragma unroll
          for (int tr = 0; tr < kTRounds; ++tr) {
            const int rr = 8 * (2 * tr + (pside ? 0 : 1));
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t ad = wb + ((c0 ^ static_cast<uint32_t>(j)) << 4) + e0 + (rr + j) * 128;
              wreg[8 * tr + j] = rr + j < R ? lds_f32(ad) + lds_f32(ad + lo_row) : 0.f;
            }
          }
        }
      }
      KWAIT(&acc_full[ast], aph);
      if (!KRP_DBG(512)) KWAIT(&oms_full[oslot], ooph);
      const uint32_t oms_s = smem_u32(smem + p.sm_ws) + static_cast<uint32_t>(oslot * kMaxTcR) * 4u;
      auto release_oms = [&]() {  // (after __syncwarp: every lane's reads of the row are done)
        if (lane == 0 && !KRP_DBG(512)) mbar_arrive(&oms_empty[oslot]);
        if (++oslot == kOmsSlots) {
          oslot = 0;
          ooph ^= 1;
        }
      };
      if (KRP_DBG(4)) {  // probe: no epilogue math
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[ast]);
        release_oms();
        if (++ast == p.NA) {
          ast = 0;
          aph ^= 1;
        }
        continue;
      }
      if (ew == 0 && lane == 0) KRP_TRACE(5, t - t0);
      tc_fence_after();
      const uint32_t tD = tbase + lane_off + p.tm_acc + ast * 2 * p.DN + (pside ? 0 : p.DN);
      const uint32_t rbuf_s = smem_u32(red + parity * (4 * R8));
      float* rbuf = red + parity * (4 * R8);
      bool released = false;
      if (active) {
        if constexpr (RA > 0) {
#pragma unroll
          for (int rnd = 0; rnd < RA / 8; ++rnd) {
            float acc8[8], z8[8];  // register copies (no pointer into Areg, which must stay in registers)
            epi_drain8(rnd, z8, tD, R, R8, p.triple);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc8[j] = Areg[8 * rnd + j];
            float w8[8];  // register copy (no pointer into wreg, which must stay in registers)
#pragma unroll
            for (int j = 0; j < 8; ++j) w8[j] = wreg[8 * (rnd >> 1) + j];
            if (!KRP_DBG(64))  // probe bit 64: drain only
            epi_math8(rnd, z8, acc8, oms_s, p.do_t && !KRP_DBG(32) && ((rnd & 1) == (pside ? 0 : 1)), w8, rbuf_s,
                      R8, sub, lane);
#pragma unroll
            for (int j = 0; j < 8; ++j) Areg[8 * rnd + j] = acc8[j];
          }
        } else {
#pragma unroll
          for (int rnd = 0; rnd < kRounds; ++rnd) {
            if (rnd < nr) {
              float acc[8];
              tmem_ld8(tA + 8 * rnd, acc);
              float w8[8];  // register copy (no pointer into wreg)
#pragma unroll
              for (int j = 0; j < 8; ++j) w8[j] = wreg[8 * (rnd >> 1) + j];
              epi_round8(rnd, acc, tD, R, R8, p.triple, oms_s, p.do_t && ((rnd & 1) == (pside ? 0 : 1)), w8,
                         rbuf_s, sub, lane);
              uint32_t accb[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) accb[j] = __float_as_uint(acc[j]);
              tmem_st8(tA + 8 * rnd, accb);
            }
          }
          tmem_st_wait();
        }
      }
      if (!released) {  // every TMEM access of this tile is done: hand the accumulator stage back
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[ast]);
      }
      release_oms();
      if (++ast == p.NA) {
        ast = 0;
        aph ^= 1;
      }
      if (p.do_t && !KRP_DBG(32)) {  // (probe bit 32: no T reduction)
        // fixed-order sum of the four lane quarters for every r (the two sides wrote disjoint rounds)
        named_bar_sync(2, kNumEpiWarps * 32);
        const int e = static_cast<int>(ew * 32 + lane);
        if (e < R) {
          const float tot = ((rbuf[e] + rbuf[R8 + e]) + rbuf[2 * R8 + e]) + rbuf[3 * R8 + e];
          p.Tpart[(pair * p.S + s) * R + e] = tot;
        }
        parity ^= 1;
      }
      if (ew == 0 && lane == 0) KRP_TRACE(6, t - t0);
      if (ew == 4 && lane == 0) KRP_TRACE(7, t - t0);
    }
    if (prev_pair >= 0)
        {  // flush the finished segment's accumulators into its partial slot
          const int kslot = static_cast<int>(blockIdx.x - cta_of_tile(prev_pair * p.S, p.T, gridDim.x));
          const int64_t slot = prev_pair * p.maxseg + kslot;
          if (threadIdx.x == kEpiWarp0 * 32) p.slot_pair[slot] = static_cast<int>(prev_pair);
          // slot layout [r][128]: for a fixed r the 32 lanes of a warp store 128 contiguous bytes
          float* dst = (pside ? p.partA1 : p.partA2) + slot * kTile * R + l;

          if constexpr (RA > 0) {
#pragma unroll
            for (int j = 0; j < RA; ++j) {
              if (active && j < R) dst[j * kTile] = Areg[j];
              Areg[j] = 0.f;
            }
          } else if (active) {
            for (int rnd = 0; rnd < nr; ++rnd) {
              float v[8];
              tmem_ld8(tA + 8 * rnd, v);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (8 * rnd + j < R) dst[(8 * rnd + j) * kTile] = v[j];
            }
          }
        }
  }
  if (threadIdx.x == kEpiWarp0 * 32) KRP_TRACE(13, 60);  // epilogue (incl. last flush) done
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tbase);
  if (threadIdx.x == 0) KRP_TRACE(13, 61);  // kernel end
}

// ------------------------------------------------------------------ reduction of partials + multi-TTVs
struct RedParams {
  int64_t M, C, S, T;
  int RB, CB, R, grid, maxseg, ldy;
  int do_p, do_q, do_t;
  uint32_t bP, bQ;            // blocks of the P and Q regions (host-computed: no 64-bit division per block)
  int nsP, nsQ, ncgP, ncgQ;   // term shares per column and column groups of each region
  int unlisted;               // test hook (KRP_ASM_UNLISTED): take the long-list path at any size
  const float *partA1, *partA2, *Tpart;
  float *Pm, *Qc, *Ts;
  float *outP, *outQ, *outT;  // non-null: the group is a single wanted mode, write its Y directly
};

// P(ρ,r) = Σ_{cb} Σ_{k < pnk[pair]} partA1[(rb*CB + cb)*maxseg + k][r][ρ%128]
// Qc(γ,r) likewise over rb;  Ts(s,r) = Σ_{pairs} Tpart[pair][s][r].
// P / Qc: one block = 32 consecutive rows (lanes: coalesced 128-byte partial reads) x 8/nsplit columns.  The
// block lists the slots its pairs used, in (o, k) order, in shared memory before the wait on the sketch
// kernel (counts from the static tile split, a warp scan places each pair's run); each column's list is split
// into nsplit contiguous shares (one warp each, 16 loads in flight, no per-term control flow: the per-term
// (o, k) bookkeeping had made the kernel issue-bound, 70 % issue-active at c4), and the shares are added in
// order: a fixed reduction order (deterministic).  nsplit grows with F = (other blocks) x maxseg so short
// term lists do not pay a block per column; region sizes come from the host (no 64-bit division).
// Ts: one block = 32 consecutive (s, r), the pair list split over the 8 warps (16 loads in flight), added in
// order.  32-bit index math throughout (the plan keeps every group and table below 2^31).
// A block never straddles a 128-row block (32 | 128) nor a region; a group with a single mode IS that
// mode's sketch, so its region is written straight into Y (outP / outQ / outT non-null).
constexpr int kRedWarps = 8;
constexpr int kAsmMaxOther = 1024;
constexpr int kAsmMaxTerms = 2048;  // listed term slots per block (8 KB of shared memory)
__host__ __device__ __forceinline__ int asm_nsplit(int64_t F) {
  return F <= 32 ? 1 : (F <= 64 ? 2 : (F <= 128 ? 4 : 8));
}
__host__ __device__ __forceinline__ int64_t asm_region_blocks(int64_t rows, int R, int64_t F) {
  const int cpb = kRedWarps / asm_nsplit(F);
  return (rows + 31) / 32 * ((R + cpb - 1) / cpb);
}
__global__ void __launch_bounds__(256, 4) tc_assemble_kernel(const __grid_constant__ RedParams p) {
  __shared__ float red[kRedWarps][32];
  __shared__ uint32_t s_term[kAsmMaxTerms];  // the used partial slots of this block's term list, in (o, k) order
  __shared__ uint32_t s_cnt[kAsmMaxOther + 1];
  const int w = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  const uint32_t bP = p.bP, bQ = p.bQ;
  uint32_t blk_id = blockIdx.x;
  if (blk_id < bP + bQ) {
    const bool rows = blk_id < bP;
    if (!rows) blk_id -= bP;
    const int nother = rows ? p.CB : p.RB;
    const int nsplit = rows ? p.nsP : p.nsQ, cpb = kRedWarps / nsplit;
    const uint32_t ncg = static_cast<uint32_t>(rows ? p.ncgP : p.ncgQ);
    const uint32_t rg = blk_id / ncg, cg = blk_id - rg * ncg;
    const uint32_t nrow = static_cast<uint32_t>(rows ? p.M : p.C);
    const uint32_t rho = rg * 32u + static_cast<uint32_t>(lane);
    const bool valid = rho < nrow;
    const uint32_t rc = valid ? rho : nrow - 1;
    const uint32_t blk = rc / kTile, l = rc % kTile;  // blk is block-uniform (32 | 128)
    const int r = static_cast<int>(cg) * cpb + w / nsplit, share = w % nsplit;
    auto pair_of = [&](uint32_t oo) {
      return rows ? blk * static_cast<uint32_t>(p.CB) + oo : oo * static_cast<uint32_t>(p.CB) + blk;
    };
    // the list of used slots (pair_of(o) * maxseg + k for k < nk(o)), formed before the wait on the sketch
    // kernel: slot counts follow from the static tile split; a block-wide scan places each pair's run
    const bool listed = !p.unlisted && nother <= kAsmMaxOther && static_cast<int64_t>(nother) * p.maxseg <= kAsmMaxTerms;
    uint32_t nterm = 0;
    if (listed) {
      for (int o = static_cast<int>(threadIdx.x); o < nother; o += blockDim.x) {
        const int64_t pr = pair_of(static_cast<uint32_t>(o));
        s_cnt[o + 1] = static_cast<uint32_t>(cta_of_tile((pr + 1) * p.S - 1, p.T, p.grid) -
                                             cta_of_tile(pr * p.S, p.T, p.grid) + 1);
      }
      __syncthreads();
      if (w == 0) {  // inclusive scan of s_cnt[1..nother] by warp 0 (32 entries per round)
        uint32_t carry = 0;
        for (int o0 = 0; o0 < nother; o0 += 32) {
          const int o = o0 + lane;
          uint32_t v = o < nother ? s_cnt[o + 1] : 0u;
#pragma unroll
          for (int m = 1; m < 32; m <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, m);
            if (lane >= m) v += u;
          }
          if (o < nother) s_cnt[o + 1] = carry + v;
          carry += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) s_cnt[0] = 0;
      }
      __syncthreads();
      for (int o = static_cast<int>(threadIdx.x); o < nother; o += blockDim.x) {
        const uint32_t b0 = s_cnt[o], n = s_cnt[o + 1] - b0;
        const uint32_t slot0 = pair_of(static_cast<uint32_t>(o)) * static_cast<uint32_t>(p.maxseg);
        for (uint32_t k = 0; k < n; ++k) s_term[b0 + k] = slot0 + k;
      }
      __syncthreads();
      nterm = s_cnt[nother];
    }
    pdl_wait();  // the partials are written by the sketch kernel
    float acc = 0.f;
    if (r < p.R) {
      const float* part = (rows ? p.partA1 : p.partA2) + static_cast<int64_t>(r) * kTile + l;
      const int64_t kstride = static_cast<int64_t>(kTile) * p.R;
      if (listed) {
        // share `share` of the used terms, 16 loads in flight, no per-term control flow
        const uint32_t f0 = static_cast<uint32_t>(share) * nterm / static_cast<uint32_t>(nsplit);
        const uint32_t f1 = static_cast<uint32_t>(share + 1) * nterm / static_cast<uint32_t>(nsplit);
        for (uint32_t f = f0; f < f1; f += 16) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            v[i] = f + i < f1 ? __ldg(part + static_cast<int64_t>(s_term[f + i]) * kstride) : 0.f;
#pragma unroll
          for (int i = 0; i < 16; ++i) acc += v[i];
        }
      } else {
        // long term lists: walk every (o, k) slot, unused slots add an exact 0
        const uint32_t F = static_cast<uint32_t>(nother) * static_cast<uint32_t>(p.maxseg);
        const uint32_t f0 = static_cast<uint32_t>(share) * F / static_cast<uint32_t>(nsplit);
        const uint32_t f1 = static_cast<uint32_t>(share + 1) * F / static_cast<uint32_t>(nsplit);
        for (uint32_t f = f0; f < f1; ++f) {
          const uint32_t o = f / static_cast<uint32_t>(p.maxseg);
          const int k = static_cast<int>(f - o * static_cast<uint32_t>(p.maxseg));
          const int64_t pr = pair_of(o);
          const int nk = cta_of_tile((pr + 1) * p.S - 1, p.T, p.grid) - cta_of_tile(pr * p.S, p.T, p.grid) + 1;
          if (k < nk) acc += __ldg(part + (pr * p.maxseg + k) * kstride);
        }
      }
    }
    red[w][lane] = acc;
    __syncthreads();
    if (share == 0 && r < p.R && valid) {
      float tot = red[w][lane];
      for (int i = 1; i < nsplit; ++i) tot += red[w + i][lane];
      float* direct = rows ? p.outP : p.outQ;
      if (direct) direct[static_cast<int64_t>(rc) * p.ldy + r] = tot;  // a single-mode group: its Y (stride ldy)
      else (rows ? p.Pm : p.Qc)[static_cast<int64_t>(rc) * p.R + r] = tot;
    }
    return;
  }
  blk_id -= bP + bQ;
  const uint32_t nT = static_cast<uint32_t>(p.S) * static_cast<uint32_t>(p.R);
  const uint32_t idx = blk_id * 32u + static_cast<uint32_t>(lane);
  pdl_wait();  // Tpart is written by the sketch kernel
  const uint32_t idc = idx < nT ? idx : nT - 1;
  const uint32_t sl = idc / static_cast<uint32_t>(p.R);
  const int r = static_cast<int>(idc - sl * static_cast<uint32_t>(p.R));
  const int64_t npairs = static_cast<int64_t>(p.RB) * p.CB;
  const int64_t p0 = w * npairs / kRedWarps, p1 = (w + 1) * npairs / kRedWarps;
  const int64_t pstride = p.S * p.R;
  const float* src = p.Tpart + static_cast<int64_t>(idc) + p0 * pstride;
  float acc = 0.f;
  for (int64_t q = p0; q < p1; q += 16, src += 16 * pstride) {  // 16 loads in flight: a share can be
    float v[16];                                                // hundreds of pairs long
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (q + i < p1) ? __ldg(src + i * pstride) : 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += v[i];
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    float tot = red[0][lane];
#pragma unroll
    for (int i = 1; i < kRedWarps; ++i) tot += red[i][lane];
    if (idx < nT) {
      if (p.outT) p.outT[static_cast<int64_t>(sl) * p.ldy + r] = tot;  // a single-mode group: its Y
      else p.Ts[idx] = tot;
    }
  }
}

int64_t assemble_blocks(int64_t M, int64_t C, int64_t S, int R, int do_p, int do_q, int do_t, int RB, int CB,
                        int maxseg) {
  return (do_p ? asm_region_blocks(M, R, static_cast<int64_t>(CB) * maxseg) : 0) +
         (do_q ? asm_region_blocks(C, R, static_cast<int64_t>(RB) * maxseg) : 0) + (do_t ? (S * R + 31) / 32 : 0);
}

struct TtvParams {
  int d, m, m2, R, ldo, ldy;
  int64_t M, C, S;
  int64_t n[kMaxD];
  int64_t gs[kMaxD];
  const float* om[kMaxD];
  const float *Pm, *Qc, *Ts;
  float* y[kMaxD];
  int want[kMaxD];
};

// Y_k(i, r) = Σ_{lin: i_k(lin) = i} src(lin, r) Π_{j in group, j != k} Ω_j(i_j(lin), r)   (fp64 sums)
// Same block shape as the assembly: 32 outputs x 8 warps splitting the o range, fixed-order combine.
__global__ void __launch_bounds__(256) tc_ttv_kernel(const __grid_constant__ TtvParams p) {
  __shared__ double red[kRedWarps][32];
  pdl_wait();  // the group objects are written by the assembly kernel
  const int w = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  int64_t blk_id = blockIdx.x;
  int k = 0;
  int64_t cnt = 0;
  for (k = 0; k < p.d; ++k) {
    if (!p.want[k]) continue;
    cnt = p.n[k] * p.R;
    const int64_t nb = (cnt + 31) / 32;
    if (blk_id < nb) break;
    blk_id -= nb;
  }
  if (k >= p.d) return;
  const int64_t idx = blk_id * 32 + lane;
  const uint32_t idc = static_cast<uint32_t>(idx < cnt ? idx : cnt - 1);
  const uint32_t i = idc / static_cast<uint32_t>(p.R);
  const int r = static_cast<int>(idc - i * static_cast<uint32_t>(p.R));
  int g0, g1;
  const float* src;
  int64_t gsize;
  if (k < p.m) {
    g0 = 0, g1 = p.m, src = p.Pm, gsize = p.M;
  } else if (k < p.m2) {
    g0 = p.m, g1 = p.m2, src = p.Qc, gsize = p.C;
  } else {
    g0 = p.m2, g1 = p.d, src = p.Ts, gsize = p.S;
  }
  const int64_t others = gsize / p.n[k];
  const int64_t o0 = w * others / kRedWarps, o1 = (w + 1) * others / kRedWarps;
  double acc = 0.0;
  for (int64_t ob = o0; ob < o1; ob += 4) {
    float xv[4], wv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      xv[u] = 0.f;
      wv[u] = 0.f;
      const int64_t o = ob + u;
      if (o < o1) {
        uint32_t rem = static_cast<uint32_t>(o), lin = i * static_cast<uint32_t>(p.gs[k]);
        float wt = 1.f;
        for (int j = g0; j < g1; ++j) {
          if (j == k) continue;
          const uint32_t nj = static_cast<uint32_t>(p.n[j]), q = rem / nj, ij = rem - q * nj;
          rem = q;
          lin += ij * static_cast<uint32_t>(p.gs[j]);
          wt *= __ldg(p.om[j] + static_cast<size_t>(ij) * p.ldo + r);
        }
        xv[u] = __ldg(src + static_cast<size_t>(lin) * p.R + r);
        wv[u] = wt;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += static_cast<double>(xv[u]) * wv[u];
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    double tot = red[0][lane];
#pragma unroll
    for (int u = 1; u < kRedWarps; ++u) tot += red[u][lane];
    if (idx < cnt) p.y[k][static_cast<size_t>(i) * p.ldy + r] = static_cast<float>(tot);
  }
}

// ------------------------------------------------------------------ host planning
struct TcPlan {
  bool ok = false;
  int m = 0, m2 = 0;
  int64_t M = 0, Mp = 0, C = 0, S = 0;  // Mp: rows as TMA sees them (M rounded up to 4 when repacked)
  bool repack = false;                  // X staged into a padded copy (row pitch not a 16-byte multiple, or
                                        // a base address that is not 16-byte aligned)
  int RB = 0, CB = 0;
  int64_t T = 0;
  int R = 0, NP = 0, N2 = 0, R8 = 0, NS = 0, NC = 0, NA = 0, CH = 16, triple = 0, DN = 0, RA = 0;
  int qh = 0;  // Q's A_hi staged in TMEM (chunk slots of 4*CH columns)
  int do_p = 0, do_q = 0, do_t = 0;
  int grid = 0, maxseg = 0, nslot = 0;
  int tm_acc = 0, tm_chunk = 0, tm_a = 0;
  uint32_t sm_x = 0, sm_bp = 0, sm_bq = 0, sm_red = 0, sm_bar = 0, sm_ws = 0, smem_bytes = 0;
};

struct DevInfo {
  int sms = 148;
  bool sm100 = false;
};
// per device (a process may drive several GPUs), computed once under a once-flag
const DevInfo& dev_info() {
  static DevInfo info[64];
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [dev] {
    DevInfo& di = info[dev];
    int major = 0, minor = 0, n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) di.sms = n;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess)
      di.sm100 = (major == 10 && minor == 0);
    cudaGetLastError();
  });
  return info[dev];
}
int num_sms() { return dev_info().sms; }
bool device_is_sm100() { return dev_info().sm100; }


// Fill geometry for a grouping (m, m2) and check the kernel's constraints.  Group sizes below 128 are
// covered by TMA's out-of-bounds zero fill (partial row / column blocks); a row pitch that is not a multiple
// of 16 bytes (M % 4 != 0) needs the padded copy (allow_repack).
bool fill_plan(const Dims& g, int R, int m, int m2, const bool* want, bool allow_repack, TcPlan& pl) {
  pl = TcPlan{};
  int64_t M = 1, C = 1, S = 1;
  for (int k = 0; k < m; ++k) M *= g.n[k];
  for (int k = m; k < m2; ++k) C *= g.n[k];
  for (int k = m2; k < g.d; ++k) S *= g.n[k];
  const bool need_repack = (M % 4) != 0;
  if (need_repack && !allow_repack) return false;
  const int64_t Mp = (M + 3) / 4 * 4;
  // the table / assembly kernels use 32-bit index math
  if (Mp * kMaxTcR >= (int64_t(1) << 31) || C * kMaxTcR >= (int64_t(1) << 31) || S * kMaxTcR >= (int64_t(1) << 31))
    return false;
  pl.Mp = Mp;
  pl.repack = need_repack;
  bool wr = false, wc = false, ws = false;
  for (int k = 0; k < g.d; ++k) {
    if (!want[k]) continue;
    if (k < m) wr = true;
    else if (k < m2) wc = true;
    else ws = true;
  }
  pl.m = m;
  pl.m2 = m2;
  pl.M = M;
  pl.C = C;
  pl.S = S;
  pl.RB = static_cast<int>((Mp + kTile - 1) / kTile);
  pl.CB = static_cast<int>((C + kTile - 1) / kTile);
  pl.T = static_cast<int64_t>(pl.RB) * pl.CB * S;
  pl.R = R;
  pl.do_t = ws ? 1 : 0;
  pl.do_p = (wr || ws) ? 1 : 0;  // T rounds alternate between z1 (P side) and z2 (Q side)
  pl.do_q = (wc || ws) ? 1 : 0;
  pl.R8 = (R + 7) / 8 * 8;
  // MMA N in steps of 8 (tcgen05, M = 128, cta_group::1: any multiple of 8 up to 256): N = R8, not round16(R)
  // (c2's R = 40: 48 -> 40 columns, sketch kernel 145.8 -> 136.1 us)
  pl.N2 = pl.R8;
  // TMEM (512 columns): NA accumulator stages of 2*DN, NC A-chunk stages of 4*CH, and A1 + A2 (2*R8) when
  // they do not live in registers.  The [hi|lo] concat form is 2 MMAs per K-step (DN = round8(R8 + R)),
  // the triple form 3 MMAs of N = N2 (DN = N2).  Large chunks amortise the split -> MMA handshake.
  {
    // qh: Q's A_hi in TMEM too (register accumulators of R8 in (48, 64] only: the QH instantiations).  At
    // R8 = 64 this is 4 slots of 4*16 columns next to the double-buffered triple-form accumulators, where
    // the TMEM-accumulator plan has 2 slots of 3*16 and holds the tile stage until the MMAs finish.
    // [rlo, rhi]: the R8 range where an option is taken by default (measured: the QH forms win at R8 = 32-64,
    // profiles/r02e_*; at R8 <= 24 the concat register plan); KRP_TC_OPT forces one (if it fits)
    struct Opt {
      int triple, na, ch, ncmin, areg, qh, rlo, rhi;
    } opts[13] = {{1, 2, 32, 2, 1, 1, 32, 48}, {1, 2, 16, 4, 1, 1, 56, 64}, {0, 2, 32, 2, 1, 0, 8, 48},
                  {1, 2, 32, 3, 1, 0, 8, 48},  {0, 2, 16, 4, 1, 0, 8, 48},  {1, 2, 32, 2, 1, 0, 8, 48},
                  {0, 2, 32, 2, 0, 0, 8, 64},  {0, 2, 16, 3, 0, 0, 8, 64},  {1, 2, 32, 2, 0, 0, 8, 64},
                  {1, 2, 16, 2, 0, 0, 8, 64},  {1, 1, 16, 2, 0, 0, 8, 64},  {0, 2, 16, 3, 1, 1, 0, 0},
                  {1, 2, 16, 3, 1, 1, 0, 0}};
    pl.NC = 0;
    const char* force = getenv("KRP_TC_OPT");  // development: force one option (if it fits)
    const int fo = force ? atoi(force) : -1;
    for (int oi = 0; oi < 13; ++oi) {
      const Opt& o = opts[oi];
      if (fo >= 0 && oi != fo) continue;
      if (fo < 0 && (pl.R8 < o.rlo || pl.R8 > o.rhi)) continue;
      if (o.areg && ((!o.qh && pl.R8 > 48) || pl.R8 > 64)) continue;  // register accumulators: R8 <= 48 (<= 64 QH)
      if (o.qh && o.ch == 32 && (pl.R8 < 24 || pl.R8 > 64 || pl.R8 == 56)) continue;  // the QH instantiations
      if (o.qh && o.ch == 16 && pl.R8 != 24 && pl.R8 != 32 && pl.R8 != 40 && pl.R8 != 56 && pl.R8 != 64) continue;
      const int dn = o.triple ? pl.N2 : (pl.R8 + R + 7) / 8 * 8;
      const int acols = o.areg ? 0 : 2 * pl.R8;
      const int slot = (o.qh ? 4 : 3) * o.ch;
      const int nc = std::min(o.ch == 16 ? 6 : 4, (512 - o.na * 2 * dn - acols) / slot);
      if (nc >= o.ncmin) {
        pl.triple = o.triple;
        pl.DN = dn;
        pl.NA = o.na;
        pl.CH = o.ch;
        pl.NC = nc;
        pl.RA = o.areg ? pl.R8 : 0;
        pl.qh = o.qh;
        break;
      }
    }
    if (pl.NC < 2 || pl.NC > kTile / pl.CH) return false;  // copies run at most one tile ahead
    pl.NP = pl.triple ? pl.R8 + pl.N2 : pl.DN;  // B-image rows (hi rows [0,R), lo rows [R8, R8+R))
  }
  pl.tm_acc = 0;
  pl.tm_chunk = pl.NA * 2 * pl.DN;
  pl.tm_a = pl.tm_chunk + pl.NC * (pl.qh ? 4 : 3) * pl.CH;
  // SMEM: X stages (64 KB each), B_P and B_Q (NP rows x 512 B each), reduction scratch, barriers
  const uint32_t bbytes = static_cast<uint32_t>(pl.NP) * 512u;
  const uint32_t misc = 2 * 4 * kMaxTcR * 4 + 256 + kOmsSlots * kMaxTcR * 4;
  const uint32_t budget = 232448 - 1024;
  int ns = static_cast<int>((budget - 2 * bbytes - misc) / (kStageFloats * 4));
  if (ns < 1) return false;
  pl.NS = std::min(ns, 3);
  pl.sm_x = 0;
  pl.sm_bp = pl.NS * kStageFloats * 4;
  pl.sm_bq = pl.sm_bp + bbytes;
  pl.sm_red = pl.sm_bq + bbytes;
  pl.sm_bar = pl.sm_red + 2 * 4 * kMaxTcR * 4;
  pl.sm_ws = pl.sm_bar + 256;
  pl.smem_bytes = pl.sm_ws + kOmsSlots * kMaxTcR * 4 + 1024;
  pl.grid = static_cast<int>(std::min<int64_t>(num_sms(), pl.T));
  // CTAs per (rb, cb) pair: a pair's S consecutive tiles meet at most ceil(S / floor(T/grid)) + 1
  // consecutive CTAs of the static split (each CTA owns >= floor(T/grid) consecutive tiles)
  {
    const int64_t per_cta = std::max<int64_t>(1, pl.T / pl.grid);
    pl.maxseg = static_cast<int>((S + per_cta - 1) / per_cta + 1);
    pl.nslot = static_cast<int>(static_cast<int64_t>(pl.RB) * pl.CB * pl.maxseg);
  }
  pl.ok = true;
  return true;
}

// Groupings that TMA can view directly are preferred; the padded copy (an extra pass over X) is used only
// when no grouping has a 16-byte row pitch, or always when force_repack (X not 16-byte aligned).
bool choose_plan(const Dims& g, int R, const bool* want, bool force_repack, TcPlan& best) {
  if (R > kMaxTcR || R < 1) return false;
  bool found = false;
  double best_cost = 1e300;
  for (int pass = 0; pass < 2 && !found; ++pass)
  for (int m = 1; m < g.d; ++m) {
    for (int m2 = m + 1; m2 <= g.d; ++m2) {
      TcPlan pl;
      if (!fill_plan(g, R, m, m2, want, pass == 1 || force_repack, pl)) continue;
      if (force_repack) pl.repack = true;
      // cost in units of one tile-GEMM: MMA work incl. ragged-tile waste, plus the per-segment
      // overhead (B operand generation + partial flush + assembly, ~8 tile-GEMMs per (rb, cb)
      // pair) — a grouping without slice modes (S = 1) makes every tile its own segment.
      const double tiles = static_cast<double>(pl.T);
      const double gemms = pl.do_p + pl.do_q;
      const double pairs = static_cast<double>(pl.RB) * pl.CB;
      const double cost = tiles * gemms * (1.0 + 0.05 * (pl.do_t ? 1 : 0)) + 8.0 * pairs * gemms;
      if (cost < best_cost) {
        best_cost = cost;
        best = pl;
        found = true;
      }
    }
  }
  return found;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

long long* g_trace_dev = nullptr;

struct WsLayout {
  size_t a1, a2, slots, tpart, pm, qc, ts, xp, total;
};
WsLayout ws_layout(const TcPlan& pl) {
  WsLayout w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  const size_t slotf = static_cast<size_t>(pl.nslot) * kTile * pl.R * sizeof(float);
  w.a1 = take(pl.do_p ? slotf : 0);
  w.a2 = take(pl.do_q ? slotf : 0);
  w.slots = take(static_cast<size_t>(pl.nslot) * sizeof(int));
  w.tpart = take(pl.do_t ? static_cast<size_t>(pl.RB) * pl.CB * pl.S * pl.R * sizeof(float) : 0);
  w.pm = take(static_cast<size_t>(pl.M) * pl.R * sizeof(float));
  w.qc = take(static_cast<size_t>(pl.C) * pl.R * sizeof(float));
  w.ts = take(static_cast<size_t>(pl.S) * pl.R * sizeof(float));
  w.xp = take(pl.repack ? static_cast<size_t>(pl.Mp) * pl.C * pl.S * sizeof(float) : 0);
  w.total = off;
  return w;
}

// Input staging for shapes TMA cannot view: Xp(ρ, rest) = X(ρ, rest) for ρ < M, 0 for M <= ρ < Mp
// (Mp = round4(M): a 16-byte row pitch); also used when X is not 16-byte aligned.  One extra pass over X.
__global__ void repack_rows_kernel(const float* __restrict__ X, int64_t M, int64_t Mp, int64_t cols,
                                   float* __restrict__ Xp) {
  const int64_t total = Mp * cols;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / Mp, r = e - c * Mp;
    Xp[e] = r < M ? X[c * M + r] : 0.f;
  }
}

size_t plan_ws_bytes(const Dims& g, int R, const bool* want) {
  size_t b = 0;
  for (int rep = 0; rep < 2; ++rep) {  // with and without the padded copy (alignment is known only at call time)
    TcPlan pl;
    if (choose_plan(g, R, want, rep == 1, pl)) b = std::max(b, ws_layout(pl).total);
  }
  return b;
}

int tc_sketch_cols(const float* X, const Dims& g, const OmegaPtrs& om, int R, int ldo, const bool* want,
                   float* const* Y, int ldy, Arena& ar, cudaStream_t s);

}  // namespace

bool tc_device_ok() { return device_is_sm100() && get_encode() != nullptr; }
void* tma_encode_fn() { return reinterpret_cast<void*>(get_encode()); }
int device_sms() { return num_sms(); }

// Columns of a KRP sketch are independent (Lemma 2.3): R > 64 runs as column groups of <= 64
// columns (one pass over X each), Ω and Y addressed through their row stride R.
size_t tc_sketch_ws_bytes(const Dims& g, int R, const bool* want) {
  size_t b = 0;
  for (int c0 = 0; c0 < R; c0 += kMaxTcR) b = std::max(b, plan_ws_bytes(g, std::min(kMaxTcR, R - c0), want));
  return b;
}

int tc_sketch(const float* X, const Dims& g, const OmegaPtrs& om, int R, const bool* want, float* const* Y, Arena& ar,
              cudaStream_t s) {
  if (!tc_device_ok()) {
    set_error("the KRP sketch needs an sm_100a device (B200) and the driver's TMA encoder");
    return KRP_EUNSUPPORTED;
  }
  for (int c0 = 0; c0 < R; c0 += kMaxTcR) {
    OmegaPtrs oc{};
    float* Yc[kMaxD] = {};
    for (int k = 0; k < g.d; ++k) {
      oc.p[k] = om.p[k] ? om.p[k] + c0 : nullptr;
      Yc[k] = (want[k] && Y[k]) ? Y[k] + c0 : nullptr;
    }
    KRP_TRY(tc_sketch_cols(X, g, oc, std::min(kMaxTcR, R - c0), R, want, Yc, R, ar, s));
  }
  return KRP_OK;
}

namespace {
int tc_sketch_cols(const float* X, const Dims& g, const OmegaPtrs& om, int R, int ldo, const bool* want,
                   float* const* Y, int ldy, Arena& ar, cudaStream_t s) {
  TcPlan pl;
  const bool misaligned = (reinterpret_cast<uintptr_t>(X) & 15u) != 0;
  if (!choose_plan(g, R, want, misaligned, pl)) {
    set_error("tcgen05 sketch: no tiling for this shape");
    return KRP_EUNSUPPORTED;
  }
  auto encode = get_encode();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return KRP_EUNSUPPORTED;
  }
  const WsLayout wl = ws_layout(pl);
  const size_t mark = ar.off;
  char* wsb = ar.take<char>(wl.total);
  if (ar.overflow()) {
    set_error("workspace too small for the tcgen05 sketch");
    return KRP_ENOMEM;
  }
  const float* Xv = X;
  if (pl.repack) {  // stage X with a 16-byte row pitch (and a 16-byte aligned base)
    float* Xp = reinterpret_cast<float*>(wsb + wl.xp);
    const int64_t total = pl.Mp * pl.C * pl.S;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(num_sms()) * 16));
    repack_rows_kernel<<<blocks, 256, 0, s>>>(X, pl.M, pl.Mp, pl.C * pl.S, Xp);
    KRP_CHECK_LAUNCH();
    Xv = Xp;
  }
  TcParams p{};
  p.M = pl.M;
  p.C = pl.C;
  p.S = pl.S;
  p.RB = pl.RB;
  p.CB = pl.CB;
  p.T = pl.T;
  p.R = R;
  p.NP = pl.NP;
  p.N2 = pl.N2;
  p.R8 = pl.R8;
  p.triple = pl.triple;
  p.DN = pl.DN;
  p.NS = pl.NS;
  p.NC = pl.NC;
  p.NA = pl.NA;
  p.do_p = pl.do_p;
  p.do_q = pl.do_q;
  p.do_t = pl.do_t;
  p.maxseg = pl.maxseg;
  p.tm_acc = pl.tm_acc;
  p.tm_chunk = pl.tm_chunk;
  p.tm_a = pl.tm_a;
  p.sm_x = pl.sm_x;
  p.sm_bp = pl.sm_bp;
  p.sm_bq = pl.sm_bq;
  p.sm_red = pl.sm_red;
  p.sm_bar = pl.sm_bar;
  p.sm_ws = pl.sm_ws;
  int64_t gs[kMaxD];  // stride of mode k inside its group (rows / cols / slices)
  {
    int64_t st = 1;
    for (int k = 0; k < pl.m; ++k) gs[k] = st, st *= g.n[k];
    st = 1;
    for (int k = pl.m; k < pl.m2; ++k) gs[k] = st, st *= g.n[k];
    st = 1;
    for (int k = pl.m2; k < g.d; ++k) gs[k] = st, st *= g.n[k];
  }
  p.partA1 = reinterpret_cast<float*>(wsb + wl.a1);
  p.partA2 = reinterpret_cast<float*>(wsb + wl.a2);
  p.slot_pair = reinterpret_cast<int*>(wsb + wl.slots);
  p.Tpart = reinterpret_cast<float*>(wsb + wl.tpart);
  float* Pm = reinterpret_cast<float*>(wsb + wl.pm);
  float* Qc = reinterpret_cast<float*>(wsb + wl.qc);
  float* Ts = reinterpret_cast<float*>(wsb + wl.ts);
  p.d = g.d;
  p.m = pl.m;
  p.m2 = pl.m2;
  p.ldo = ldo;
  for (int k = 0; k < kMaxD; ++k) {
    p.om[k] = k < g.d ? om.p[k] : nullptr;
    p.gn[k] = k < g.d ? static_cast<uint32_t>(g.n[k]) : 1u;
    p.ggs[k] = k < g.d ? static_cast<uint32_t>(gs[k]) : 1u;
  }
  {
    const char* e = getenv("KRP_TC_DEBUG");
    p.dbg = e ? atoi(e) : 0;
    const char* w = getenv("KRP_TC_WAIT_NS");
    p.wait_ns = w ? static_cast<uint32_t>(atol(w)) : 10000000u;
    const char* ms = getenv("KRP_TC_MMA_SPIN");
    p.mma_spin = ms ? atoi(ms) : 1;  // measured: c4 -9 %, c2 -1 % (profiles/r01f_ab_mma_spin.log)
    const char* ss = getenv("KRP_TC_SPLIT_SPIN");
    p.split_spin = ss ? atoi(ss) : 1;
    p.trace = nullptr;
    if (getenv("KRP_TC_TRACE")) {
      static long long* tr = nullptr;
      if (!tr) cudaMalloc(&tr, 16 * 64 * sizeof(long long));
      cudaMemsetAsync(tr, 0, 16 * 64 * sizeof(long long), s);
      p.trace = tr;
    }
  }

  CUtensorMap tmap;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(pl.Mp), static_cast<cuuint64_t>(pl.C),
                          static_cast<cuuint64_t>(pl.S)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(pl.Mp) * 4, static_cast<cuuint64_t>(pl.Mp * pl.C) * 4};
    cuuint32_t box[3] = {32, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(Xv), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
      return KRP_ECUDA;
    }
  }
  // 1. the fused tile kernel (the Khatri-Rao rows are formed on chip)
  using KernFn = void (*)(const CUtensorMap, const TcParams);
  // register-accumulator variants are sized to R8 exactly (register pressure), all with CH = 32
  KernFn kern = nullptr;
  if (pl.qh && pl.CH == 32) {
    switch (pl.RA) {
      case 24: kern = krp_tc_sketch_kernel<32, 24, true>; break;
      case 32: kern = krp_tc_sketch_kernel<32, 32, true>; break;
      case 40: kern = krp_tc_sketch_kernel<32, 40, true>; break;
      case 48: kern = krp_tc_sketch_kernel<32, 48, true>; break;
      case 64: kern = krp_tc_sketch_kernel<32, 64, true>; break;  // (development A/B at c5)
      default: set_error("tcgen05 sketch: no QH instantiation for CH = 32, R8 = %d", pl.RA); return KRP_EUNSUPPORTED;
    }
  } else if (pl.qh) {
    switch (pl.RA) {
      case 24: kern = krp_tc_sketch_kernel<16, 24, true>; break;
      case 32: kern = krp_tc_sketch_kernel<16, 32, true>; break;
      case 40: kern = krp_tc_sketch_kernel<16, 40, true>; break;
      case 56: kern = krp_tc_sketch_kernel<16, 56, true>; break;
      case 64: kern = krp_tc_sketch_kernel<16, 64, true>; break;
      default: set_error("tcgen05 sketch: no QH instantiation for R8 = %d", pl.RA); return KRP_EUNSUPPORTED;
    }
  } else if (pl.RA == 0) {
    kern = pl.CH == 32 ? krp_tc_sketch_kernel<32, 0> : krp_tc_sketch_kernel<16, 0>;
  } else {
    const bool c32 = pl.CH == 32;
    switch (pl.RA) {
      case 8: kern = c32 ? krp_tc_sketch_kernel<32, 8> : krp_tc_sketch_kernel<16, 8>; break;
      case 16: kern = c32 ? krp_tc_sketch_kernel<32, 16> : krp_tc_sketch_kernel<16, 16>; break;
      case 24: kern = c32 ? krp_tc_sketch_kernel<32, 24> : krp_tc_sketch_kernel<16, 24>; break;
      case 32: kern = c32 ? krp_tc_sketch_kernel<32, 32> : krp_tc_sketch_kernel<16, 32>; break;
      case 40: kern = c32 ? krp_tc_sketch_kernel<32, 40> : krp_tc_sketch_kernel<16, 40>; break;
      default: kern = c32 ? krp_tc_sketch_kernel<32, 48> : krp_tc_sketch_kernel<16, 48>; break;
    }
  }
  KRP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(pl.smem_bytes)));
  prof_begin(s);
#if KRP_SKETCH_PDL
  KRP_CHECK_CUDA(launch_pdl(kern, dim3(pl.grid), dim3(kThreads), pl.smem_bytes, s, tmap, p));
#else
  // a plain launch: the kernel reads X and the Ω_k, which the work before it in the stream may write
  kern<<<pl.grid, kThreads, pl.smem_bytes, s>>>(tmap, p);
#endif
  KRP_CHECK_LAUNCH();
  prof_end(s, 4.0 * static_cast<double>(g.N), 2.0 * static_cast<double>(g.N) * R * (pl.do_p + pl.do_q));
  if (p.trace) {  // development: dump CTA 0's role timeline (KRP_TC_TRACE=<file>)
    long long h[16 * 64];
    cudaMemcpyAsync(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (FILE* f = fopen(getenv("KRP_TC_TRACE"), "w")) {
      for (int i = 0; i < 16 * 64; ++i) fprintf(f, "%lld%c", h[i], (i % 64 == 63) ? '\n' : ' ');
      fclose(f);
    }
  }
  // 2. fixed-order sum of the per-CTA partials, then the multi-TTVs of the three groups
  {
    RedParams rp{};
    rp.M = pl.M;
    rp.C = pl.C;
    rp.S = pl.S;
    rp.T = pl.T;
    rp.RB = pl.RB;
    rp.CB = pl.CB;
    rp.R = R;
    rp.grid = pl.grid;
    rp.maxseg = pl.maxseg;
    rp.ldy = ldy;
    rp.do_p = pl.do_p;
    rp.do_q = pl.do_q;
    rp.do_t = pl.do_t;
    rp.partA1 = p.partA1;
    rp.partA2 = p.partA2;
    rp.Tpart = p.Tpart;
    rp.Pm = Pm;
    rp.Qc = Qc;
    rp.Ts = Ts;
    rp.outP = (pl.m == 1 && want[0]) ? Y[0] : nullptr;
    rp.outQ = (pl.m2 - pl.m == 1 && want[pl.m]) ? Y[pl.m] : nullptr;
    rp.outT = (g.d - pl.m2 == 1 && want[pl.m2]) ? Y[pl.m2] : nullptr;
    if (rp.do_t && pl.RB * pl.CB == 1 && !rp.outT) {
      // one (row block, col block) pair: the per-tile T rows already are Ts (same [s][r] layout), so the
      // multi-TTV reads them in place and the assembly skips the slice region
      Ts = p.Tpart;
      rp.do_t = 0;
    }
    {
      const int64_t FP = static_cast<int64_t>(pl.CB) * pl.maxseg, FQ = static_cast<int64_t>(pl.RB) * pl.maxseg;
      rp.nsP = asm_nsplit(FP);
      rp.nsQ = asm_nsplit(FQ);
      rp.ncgP = (R + kRedWarps / rp.nsP - 1) / (kRedWarps / rp.nsP);
      rp.ncgQ = (R + kRedWarps / rp.nsQ - 1) / (kRedWarps / rp.nsQ);
      rp.bP = static_cast<uint32_t>(rp.do_p ? asm_region_blocks(pl.M, R, FP) : 0);
      rp.bQ = static_cast<uint32_t>(rp.do_q ? asm_region_blocks(pl.C, R, FQ) : 0);
      const char* ul = getenv("KRP_ASM_UNLISTED");
      rp.unlisted = ul && ul[0] == '1';
    }
    const int64_t nblk = assemble_blocks(pl.M, pl.C, pl.S, R, rp.do_p, rp.do_q, rp.do_t, pl.RB, pl.CB, pl.maxseg);
    KRP_CHECK_CUDA(launch_pdl(tc_assemble_kernel, dim3(static_cast<unsigned>(nblk)), dim3(256), 0, s, rp));
    KRP_CHECK_LAUNCH();
  }
  {
    TtvParams tv{};
    tv.d = g.d;
    tv.m = pl.m;
    tv.m2 = pl.m2;
    tv.R = R;
    tv.ldo = ldo;
    tv.ldy = ldy;
    tv.M = pl.M;
    tv.C = pl.C;
    tv.S = pl.S;
    int64_t nout = 0;
    for (int k = 0; k < g.d; ++k) {
      tv.n[k] = g.n[k];
      tv.gs[k] = gs[k];
      tv.om[k] = om.p[k];
      // single-mode groups were written by the assembly
      const bool single = (k < pl.m) ? (pl.m == 1) : (k < pl.m2 ? (pl.m2 - pl.m == 1) : (g.d - pl.m2 == 1));
      tv.want[k] = (want[k] && !single) ? 1 : 0;
      tv.y[k] = tv.want[k] ? Y[k] : nullptr;
      if (tv.want[k]) nout += (g.n[k] * R + 31) / 32;
    }
    tv.Pm = Pm;
    tv.Qc = Qc;
    tv.Ts = Ts;
    if (nout > 0) {
      KRP_CHECK_CUDA(launch_pdl(tc_ttv_kernel, dim3(static_cast<unsigned>(nout)), dim3(256), 0, s, tv));
      KRP_CHECK_LAUNCH();
    }
  }
  ar.off = mark;
  return KRP_OK;
}

}  // namespace
}  // namespace krp
