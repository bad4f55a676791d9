// krp_sketch_tc.cu — the fused KRP sketch on sm_100a tensor cores (3xTF32), role-specialised CTA pairs.
//
// Method (Alg. 7 line 3 with memoization).  Split the modes into
// rows [0,m), cols [m,m2) and slices [m2,d); X is then an M x C x S array (first index
// fastest, a free reshape).  With the Khatri-Rao rows W_L(ρ,r) = Π_{k<m} Ω_k(i_k(ρ),r),
// W_R(γ,r) = Π_{m<=k<m2} Ω_k(i_k(γ),r) and Ω_S(s,r) = Π_{k>=m2} Ω_k(i_k(s),r), every Y_n is a
// multi-TTV of one of three small objects:
//     A1(ρ,r) = Σ_s Ω_S(s,r) Σ_γ X(ρ,γ,s) W_R(γ,r)            -> row modes     ("P side")
//     A2(γ,r) = Σ_s Ω_S(s,r) Σ_ρ X(ρ,γ,s) W_L(ρ,r)            -> col modes     ("Q side")
//     T(s,r)  = Σ_ρ W_L(ρ,r) Σ_γ X(ρ,γ,s) W_R(γ,r)            -> slice modes   (either side)
// (4·N·R flops for all modes; every element of X is read from HBM once).
//
// Tiles are 128 x 128 blocks X(ρ-block, γ-block, s), loaded by TMA (four SWIZZLE_128B boxes of
// {32 ρ, 128 γ}).  The two contractions of a tile run on tcgen05 in 3xTF32 (x = hi + lo, hi = x
// truncated to tf32 — what the tensor core reads — lo = x - hi exact in fp32; products hi·hi + hi·lo +
// lo·hi, fp32 accumulation in TMEM):
//     P role:  z1 = X_tile · W_R(γ-block)     (MMA M = ρ, K = γ; A = the tile, transposed into TMEM)
//     Q role:  z2 = X_tileᵀ · W_L(ρ-block)    (MMA M = γ, K = ρ; A_hi = the raw tile in SMEM, K-major)
// A CTA does ONE role.  When a sketch needs both sides, CTAs come in pairs (a 2-CTA cluster, P = rank 0,
// Q = rank 1) that walk the same tile sequence; each CTA issues two of the four TMA boxes of a tile with
// .multicast::cluster, so the tile is read from L2 once and lands in both CTAs' shared memory.  Giving each
// CTA one side halves its TMEM and SMEM needs (one B operand, one accumulator pair), which buys 4 chunk
// slots between the split warps and the MMA issuer and 2-3 tile stages.
//
// B operands: the Khatri-Rao rows of the role's K block (P: W_R of the γ-block, Q: W_L of the ρ-block) are
// formed from the Ω_k by the epilogue warps at every (ρ-block, γ-block) segment start, split hi/lo and
// written straight into shared memory in the UMMA K-major SWIZZLE_128B layout [k-atom][2·R8 rows][128 B]
// (rows [0,R8) hi, [R8,2·R8) lo); they are never materialised in global memory.
//
// Per tile (one role):  the split warps copy the tile into TMEM chunks of 32 K columns (P: hi and lo with
// lane = ρ — the transpose; Q: lo with lane = γ, optionally hi too); the MMA warp issues
// hi × [B_hi | B_lo] (N = 2·R8) and lo × B_hi (N = round16(R)) per K-step of 8; the epilogue warps drain
// z = D[r] + D[R8 + r], accumulate A += z·Ω_S(s) in registers, and (T role) form T(s,r) = Σ_lanes z·W by a
// 32-lane butterfly + a fixed-order cross-warp sum.  Per-(segment, CTA pair) partials of A go to a workspace
// slot; tc_assemble_kernel sums them in a fixed order (no float atomics: deterministic results).
//
// Warp roles (640 threads): 0-7 split (two per TMEM lane quarter, alternating chunks), 8-15 epilogue
// (lane quarter x round parity), 16 TMA producer, 17 MMA issuer, 18-19 idle.
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

constexpr int kNumSplitWarps = 8;  // WG0-1: two per TMEM lane quarter, alternating chunks
constexpr int kEpiWarp0 = 8;
constexpr int kNumEpiWarps = 16;   // WG2-5: four per TMEM lane quarter (rounds rnd = hq + 4i)
constexpr int kTmaWarp = 24;       // WG6: TMA producer, MMA issuer, 2 idle
constexpr int kMmaWarp = 25;
constexpr int kThreads = 28 * 32;
// launch budget 72 registers/thread (64K / 896); setmaxnreg moves them: 256*(72-64) + 128*(72-24) = 512*(88-72)
constexpr int kRegsSplit = 64, kRegsEpi = 88, kRegsProd = 24;
constexpr int kTile = 128;
constexpr int kCH = 32;                        // K columns per split -> MMA chunk
constexpr int kNkc = kTile / kCH;              // chunks per tile
constexpr int kStageBytes = 4 * 128 * 32 * 4;  // one 128 x 128 fp32 tile = 4 TMA boxes of {32, 128}
constexpr int kMaxTcR = 64;                    // columns per launch (wider R: column groups, krp_sketch_tc host)
constexpr int kNA = 2;                         // accumulator stages
enum { kRoleP = 0, kRoleQ = 1, kTBoth = 2 };  // t_role: P, Q, or split between the pair

struct TcParams {
  int64_t M, C, S;  // group sizes: rows (modes [0,m)), cols ([m,m2)), slices ([m2,d))
  int RB, CB;
  int64_t T;        // tiles, order (rb, cb, s) with s fastest
  int R, R8, N2, DN;  // DN = 2*R8: accumulator columns = B-image rows
  int ldo;            // row stride of the Ω_k (floats)
  int NS;
  int NC[2], ccols[2];  // per role: chunk slots, TMEM columns per slot
  int pairs, clustered, role_fixed, t_role, qhi_tmem;
  int do_a[2];          // per role: accumulate A (the group's modes are wanted)
  int ncl, maxseg;      // tile groups (CTA pairs or CTAs); max groups touching one (rb, cb) pair
  int tm_acc, tm_chunk;
  uint32_t sm_b, sm_red, sm_oms, sm_bar;
  float* part[2];  // per role: [npairs*maxseg][R][128] partial A1 (P) / A2 (Q)
  float* Tpart;    // [RB*CB][S][R]
  int d, m, m2;
  int64_t n[kMaxD], gs[kMaxD];  // mode sizes; stride of mode k inside its group
  const float* om[kMaxD];       // Ω_k (null: not given — the wanted mode of a single-mode sketch)
  long long* trace;             // development timeline (KRP_DEV_TRACE builds only)
};

// floor(num / den) for 0 <= num < 2^62, den > 0, without the 64-bit integer division routine
__host__ __device__ __forceinline__ int64_t fdiv64(int64_t num, int64_t den) {
  int64_t q = static_cast<int64_t>(static_cast<double>(num) / static_cast<double>(den));
  while (q * den > num) --q;
  while ((q + 1) * den <= num) ++q;
  return q;
}
// tile group owning tile t under the static split a0(b) = floor(b*T/ngrp): the largest b with a0(b) <= t
__host__ __device__ __forceinline__ int grp_of_tile(int64_t t, int64_t T, int ngrp) {
  return static_cast<int>(fdiv64((t + 1) * ngrp - 1, T));
}

__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }
__device__ __forceinline__ float lds_f32(uint32_t saddr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t saddr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(saddr), "f"(v) : "memory");
}

// Khatri-Rao row values W(lin, r0 + j), j < NJ, of a linear index inside the group [g0, g1):
// W = Π_k Ω_k(i_k(lin), r) with i_k = (lin / gs[k]) % n[k]; columns r >= R are 0.  The NJ loads of one mode
// are independent (issued back to back), so a row costs one load latency per mode.  Ω_k that are not given
// (null) are skipped: they never reach the wanted Y.
template <int NJ>
__device__ __forceinline__ void kr_row(const TcParams& p, int g0, int g1, uint32_t lin, int r0, int R, float (&w)[NJ]) {
#pragma unroll
  for (int j = 0; j < NJ; ++j) w[j] = r0 + j < R ? 1.f : 0.f;
  for (int k = g0; k < g1; ++k) {
    if (!p.om[k]) continue;
    const uint32_t ik = (lin / static_cast<uint32_t>(p.gs[k])) % static_cast<uint32_t>(p.n[k]);
    const float* row = p.om[k] + static_cast<size_t>(ik) * p.ldo + r0;
    float v[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) v[j] = r0 + j < R ? __ldg(row + j) : 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) w[j] *= v[j];
  }
}

// Ω_S(s, c) for this lane's two columns c = lane, lane + 32 (R <= 64), prefetched one tile ahead: the
// loads of up to kOmsDefer slice modes are only issued here (their product is formed when the row is
// stored, a tile later, so no warp waits on them); further slice modes are multiplied in immediately.
constexpr int kOmsDefer = 3;
struct OmsPrefetch {
  float v[kOmsDefer][2];  // raw loads of the first kOmsDefer slice modes (consumed a tile later)
  float x0, x1;           // product of further slice modes (rare; formed immediately)
};
__device__ __forceinline__ void oms_fetch(const TcParams& p, uint32_t s, uint32_t lane, int R, OmsPrefetch& f) {
  const int c0 = static_cast<int>(lane), c1 = c0 + 32;
  const bool one = p.d - p.m2 == 1;
#pragma unroll
  for (int q = 0; q < kOmsDefer; ++q) {
    const int k = p.m2 + q;
    f.v[q][0] = 1.f;
    f.v[q][1] = 1.f;
    if (k < p.d && p.om[k]) {
      const uint32_t ik = one ? s : (s / static_cast<uint32_t>(p.gs[k])) % static_cast<uint32_t>(p.n[k]);
      const float* row = p.om[k] + static_cast<size_t>(ik) * p.ldo;
      if (c0 < R) f.v[q][0] = __ldg(row + c0);
      if (c1 < R) f.v[q][1] = __ldg(row + c1);
    }
  }
  f.x0 = 1.f;
  f.x1 = 1.f;
  for (int k = p.m2 + kOmsDefer; k < p.d; ++k) {
    if (!p.om[k]) continue;
    const uint32_t ik = (s / static_cast<uint32_t>(p.gs[k])) % static_cast<uint32_t>(p.n[k]);
    const float* row = p.om[k] + static_cast<size_t>(ik) * p.ldo;
    if (c0 < R) f.x0 *= __ldg(row + c0);
    if (c1 < R) f.x1 *= __ldg(row + c1);
  }
}

// every non-hot wait: try_wait with a 10 ms suspend-time hint
#define KWAIT(bar, par) mbar_wait_hint((bar), (par), 10000000u)

// Development timeline (-DKRP_DEV_TRACE, KRP_TC_TRACE=<file>): CTAs 0 and 1 record %globaltimer (ns) at
// per-tile role events; compiled out of production builds.
#ifndef KRP_SPLIT_SPIN
#define KRP_SPLIT_SPIN 1
#endif
#ifndef KRP_MMA_SPIN
#define KRP_MMA_SPIN 1
#endif
#define SPLIT_WAIT(bar, par) \
  do { if (KRP_SPLIT_SPIN) mbar_wait_spin((bar), (par)); else KWAIT((bar), (par)); } while (0)
#define MMA_WAIT(bar, par) \
  do { if (KRP_MMA_SPIN) mbar_wait_spin((bar), (par)); else KWAIT((bar), (par)); } while (0)
#ifndef KRP_PF_DIST
#define KRP_PF_DIST 3
#endif
#ifdef KRP_DEV_TRACE
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define KRP_TRACE(slot, idx)                                                                        \
  do {                                                                                              \
    if (p.trace && blockIdx.x < 2 && (idx) < 64) p.trace[(blockIdx.x * 16 + (slot)) * 64 + (idx)] = gtimer(); \
  } while (0)
#define KRP_SEC_BEGIN() long long sec_t0_ = clock64()
#define KRP_SEC(i)                                \
  do {                                            \
    const long long n_ = clock64();               \
    sec_acc_[i] += n_ - sec_t0_;                  \
    sec_t0_ = n_;                                 \
  } while (0)
#else
#define KRP_TRACE(slot, idx) \
  do {                       \
  } while (0)
#define KRP_SEC_BEGIN() \
  do {                  \
  } while (0)
#define KRP_SEC(i) \
  do {             \
  } while (0)
#endif

// Transposed 32-lane butterfly of 8 per-lane values: afterwards lanes 4c..4c+3 hold Σ_lanes tv[c]
// (3 halving levels + 2 plain levels: 9 shuffles for 8 columns).
__device__ __forceinline__ float butterfly8(float (&tv)[8], uint32_t lane) {
#pragma unroll
  for (int lvl = 0; lvl < 3; ++lvl) {
    const int msk = 16 >> lvl;
    const int h = 4 >> lvl;
    const bool upper = (lane & msk) != 0;
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const float send = upper ? tv[j] : tv[j + h];
      const float keep = upper ? tv[j + h] : tv[j];
      tv[j] = keep + __shfl_xor_sync(0xffffffffu, send, msk);
    }
  }
  tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 2);
  tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 1);
  return tv[0];
}

// Synchronisation (mbarriers; chunk g of the CTA sits in slot g % NC):
//   full_x[st]      tile stage st landed                        (own producer's expect_tx + 64 KB of TMA bytes)
//   empty_x[st]     stage st may be overwritten                  (split warps [+ the Q MMA commit], of both CTAs
//                                                                  of a cluster)
//   chunk_ready[c]  chunk slot c is free (its MMAs are done)     (1 MMA commit; split waits)
//   chunk_full[c]   split wrote the chunk                        (4 split warps of one parity; MMA waits)
//   acc_full[a]     accumulator stage a complete                 (1 MMA commit; epilogue waits)
//   acc_empty[a]    epilogue drained accumulator stage a         (8 epilogue warps; MMA waits)
//   b_ready         the segment's B image is in shared memory   (1 epilogue arrival; MMA waits)
struct KBars {
  uint64_t *full_x, *empty_x, *chunk_full, *chunk_ready, *acc_full, *acc_empty, *b_ready;
};

// ------------------------------------------------------------------ split warps: tile -> TMEM (hi / lo)
// P (lane = ρ): scalar shared loads (the transpose), hi = the raw value, lo = x - tf32(x).
// Q (lane = γ): 16-byte loads along ρ; lo (and hi when QHI) to TMEM.
template <int ROLE, bool QHI>
__device__ __forceinline__ void split_loop(const TcParams& p, const KBars& kb, uint32_t smem0, uint32_t tbase,
                                           int ntile, int NC, int ccols, int rank, uint32_t warp, uint32_t lane) {
  const uint32_t sub = warp & 3;
  const int par = static_cast<int>(warp >> 2);  // this warp takes chunks kc % 2 == par
  const uint32_t chunk0 = tbase + ((32u * sub) << 16) + static_cast<uint32_t>(p.tm_chunk);
  constexpr uint32_t kLoOff = (ROLE == kRoleP || QHI) ? kCH : 0;
  // P view: element (ρ = 32*sub + lane, γ) of box `sub` at byte γ*128 + (((lane>>2) ^ (γ&7)) << 4) + (lane&3)*4
  uint32_t base8[8];
  if constexpr (ROLE == kRoleP) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      base8[j] = smem0 + sub * 16384u + ((((lane >> 2) ^ static_cast<uint32_t>(j)) << 4) | ((lane & 3u) << 2)) +
                 static_cast<uint32_t>(j) * 128u;
  } else {
    // Q view: row γ = 32*sub + lane of box kc (32 ρ, 8 chunks of 16 B swizzled by γ & 7)
    const uint32_t gq = 32 * sub + lane;
#pragma unroll
    for (int j = 0; j < 8; ++j) base8[j] = smem0 + gq * 128u + ((static_cast<uint32_t>(j) ^ (gq & 7u)) << 4);
  }
  const uint32_t peer_empty0 =
      p.clustered ? mapa_shared(smem_u32(kb.empty_x), static_cast<uint32_t>(rank ^ 1)) : 0u;
  const int NS = p.NS;
  int xst = 0;
  uint32_t xph = 0;
  // chunk g of the CTA (all tiles) sits in slot g % NC; this warp takes g % 2 == par (kNkc is even)
  int cst = par % NC;
  uint32_t cph = par >= NC ? 1u : 0u;
  for (int it = 0; it < ntile; ++it) {
    if (warp == 0 && lane == 0) KRP_TRACE(4, it);
    KWAIT(&kb.full_x[xst], xph);
    if (warp == 0 && lane == 0) KRP_TRACE(5, it);
    const uint32_t stage_off = static_cast<uint32_t>(xst) * kStageBytes;
#pragma unroll
    for (int kk = 0; kk < kNkc / 2; ++kk) {
      const int kc = 2 * kk + par;
      SPLIT_WAIT(&kb.chunk_ready[cst], cph ^ 1);
      tc_fence_after();
      const uint32_t ch = chunk0 + static_cast<uint32_t>(cst * ccols);
      uint32_t v[kCH];
      if constexpr (ROLE == kRoleP) {
        const uint32_t goff = stage_off + static_cast<uint32_t>(kc) * (kCH * 128u);
#pragma unroll
        for (int j = 0; j < kCH; ++j) v[j] = __float_as_uint(lds_f32(base8[j & 7] + goff + static_cast<uint32_t>(j & ~7) * 128u));
        tmem_st<kCH>(ch, v);  // hi: the raw value (the tensor core truncates to tf32)
      } else {
        const uint32_t goff = stage_off + static_cast<uint32_t>(kc) * 16384u;
#pragma unroll
        for (int qq = 0; qq < kCH / 4; ++qq) {
          float a0, a1, a2, a3;
          lds_v4(base8[qq] + goff, a0, a1, a2, a3);
          v[4 * qq] = __float_as_uint(a0), v[4 * qq + 1] = __float_as_uint(a1);
          v[4 * qq + 2] = __float_as_uint(a2), v[4 * qq + 3] = __float_as_uint(a3);
        }
        if constexpr (QHI) tmem_st<kCH>(ch, v);
      }
#pragma unroll
      for (int j = 0; j < kCH; j += 2) {
        const float2 x = make_float2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
        const float2 lo = f2_sub(x, make_float2(__uint_as_float(tf32_hi_bits(x.x)), __uint_as_float(tf32_hi_bits(x.y))));
        v[j] = __float_as_uint(lo.x);
        v[j + 1] = __float_as_uint(lo.y);
      }
      tmem_st<kCH>(ch + kLoOff, v);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&kb.chunk_full[cst]);
      cst += 2;  // skip the other parity's chunk (NC >= 2: at most one wrap)
      if (cst >= NC) {
        cst -= NC;
        cph ^= 1;
      }
    }
    __syncwarp();
    if (warp == 0 && lane == 0) KRP_TRACE(6, it);
    if (warp == 4 && lane == 0) KRP_TRACE(7, it);
    if (lane == 0) {
      mbar_arrive(&kb.empty_x[xst]);
      if (p.clustered) mbar_arrive_cluster(peer_empty0 + static_cast<uint32_t>(xst) * 8u);
    }
    if (++xst == NS) {
      xst = 0;
      xph ^= 1;
    }
  }
}

// B image of one segment: rows [0,R8) hi, [R8, 2R8) lo of W(kblk*128 + k, r) in the UMMA K-major SWIZZLE_128B
// layout [k-atom][2*R8 rows][128 B]; zero outside the group.  256 epilogue threads: k = e % 128, column half e / 128.
__device__ __forceinline__ void gen_bimage(const TcParams& p, uint32_t bimg_s, int kg0, int kg1, uint32_t kgsize, int kblk,
                                        int R, int R8, int DN, uint32_t ew, uint32_t lane) {
  const int e = static_cast<int>(ew * 32 + lane);  // 0..511
  const int k = e & 127, r0 = (e >> 7) * 16;      // K row k, 16 columns [r0, r0 + 16)
  if (r0 >= R8) return;
  const uint32_t lin = static_cast<uint32_t>(kblk) * kTile + static_cast<uint32_t>(k);
  const bool inb = lin < kgsize;
  const uint32_t base = bimg_s + static_cast<uint32_t>(k >> 5) * (DN * 128u) + (k & 3u) * 4u;
  const uint32_t k8 = (static_cast<uint32_t>(k) & 31u) >> 2;
  float w[16];
  kr_row<16>(p, kg0, kg1, lin, r0, inb ? R : 0, w);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int r = r0 + j;
    if (r < R8) {
      const float whi = __uint_as_float(tf32_hi_bits(w[j]));
      const uint32_t rh = static_cast<uint32_t>(r), rl = static_cast<uint32_t>(R8 + r);
      sts_f32(base + rh * 128u + ((k8 ^ (rh & 7u)) << 4), whi);
      sts_f32(base + rl * 128u + ((k8 ^ (rl & 7u)) << 4), w[j] - whi);
    }
  }
}

// ------------------------------------------------------------------ epilogue warps
// Per tile: z = D[r] + D[R8 + r] (columns >= R are exactly zero: the B image rows r >= R are zero),
// A += z·Ω_S(s) in registers, and on T rounds the 32-lane butterfly of z·W into the quarter's T scratch,
// then (after the accumulator is handed back) a fixed-order sum of the four quarters -> Tpart.
// RH: rounds per thread (rounds rnd = hq + 4i, i < RH, 8 columns each).  DOA: this role's A is wanted.
// TT: which warps do T — 0 none, 1 warps with even hq (even rounds), 2 odd hq (the pair splits T between its
// roles: P the even, Q the odd rounds), 3 all.
template <int RH, bool DOA, int TT>
__device__ __forceinline__ void epi_loop(const TcParams& p, const KBars& kb, uint8_t* smem, uint32_t tbase, int role,
                                         int grp, int64_t t0, int64_t t1, uint32_t warp, uint32_t lane) {
  const uint32_t ew = warp - kEpiWarp0;      // 0..15
  const uint32_t sub = warp & 3;             // TMEM lane quarter
  const int hq = static_cast<int>(ew >> 2);  // this warp's rounds: rnd % 4 == hq
  const int l = static_cast<int>(32 * sub + lane);
  const int R = p.R, R8 = p.R8, DN = p.DN;
  const int nval = (R8 / 8 - hq + 3) / 4;  // valid rounds of this warp (rnd < R8 / 8)
  const bool t_warp = TT == 3 || (TT == 1 && (hq & 1) == 0) || (TT == 2 && (hq & 1) == 1);
  const int t_threads = TT == 3 ? kNumEpiWarps * 32 : kNumEpiWarps * 16;  // warps in the T barrier
  const int ngrp = p.ncl;
  // this role's K group (B image) and, for T, the M group (the lane's own Khatri-Rao row)
  const int kg0 = role == kRoleP ? p.m : 0, kg1 = role == kRoleP ? p.m2 : p.m;
  const int mg0 = role == kRoleP ? 0 : p.m, mg1 = role == kRoleP ? p.m : p.m2;
  const uint32_t kgsize = static_cast<uint32_t>(role == kRoleP ? p.C : p.M);
  const uint32_t mgsize = static_cast<uint32_t>(role == kRoleP ? p.M : p.C);
  uint8_t* bimg = smem + p.sm_b;
  float* red = reinterpret_cast<float*>(smem + p.sm_red);  // [2 parities][4 lane quarters][64]
  float* oms_w = reinterpret_cast<float*>(smem + p.sm_oms) + ew * 64;
  const uint32_t oms_s = smem_u32(oms_w);
  const uint32_t tacc = tbase + ((32u * sub) << 16) + static_cast<uint32_t>(p.tm_acc);
  const uint32_t rbuf0 = smem_u32(red + sub * 64);
  const int64_t S = p.S;
  const int CB = p.CB;
  float A[RH * 8], W[RH * 8];
#pragma unroll
  for (int j = 0; j < RH * 8; ++j) A[j] = 0.f, W[j] = 0.f;
  OmsPrefetch om_nx;  // Ω_S row of the next tile (this lane's two columns)
  // one slice mode (the common case): Ω_S(s, c) = Ω_{m2}(s, c); the row base and the lane's column predicates
  // are fixed for the whole loop (no per-tile parameter loads or index decomposition)
  const bool one_slice = p.d - p.m2 == 1 && p.om[p.m2] != nullptr;
  const float* oms_base = one_slice ? p.om[p.m2] + lane : nullptr;
  const int ldo = p.ldo;
  const bool c0ok = static_cast<int>(lane) < R, c1ok = static_cast<int>(lane) + 32 < R;
#define KRP_OMS_FETCH(snext)                                                      \
  do {                                                                            \
    if (one_slice) {                                                              \
      const float* row_ = oms_base + static_cast<size_t>(snext) * ldo;            \
      om_nx.v[0][0] = c0ok ? __ldg(row_) : 0.f;                                   \
      om_nx.v[0][1] = c1ok ? __ldg(row_ + 32) : 0.f;                              \
    } else {                                                                      \
      oms_fetch(p, static_cast<uint32_t>(snext), lane, R, om_nx);                 \
    }                                                                             \
  } while (0)
  if (one_slice) {
#pragma unroll
    for (int q = 0; q < kOmsDefer; ++q) om_nx.v[q][0] = om_nx.v[q][1] = 1.f;
    om_nx.x0 = om_nx.x1 = 1.f;
  }
  if (DOA && t0 < t1) KRP_OMS_FETCH(t0 % S);
  int ast = 0;
  uint32_t aph = 0;
  int64_t prev_pair = -1;
  int parity = 0;
  int64_t pair = t0 / S, s = t0 % S;
  // the finished segment's accumulators -> its partial slot ([r][128]: a warp stores 128 B per r)
#define KRP_FLUSH(fpair)                                                        \
  do {                                                                          \
    const int kslot = grp - grp_of_tile((fpair) * S, p.T, ngrp);                \
    const int64_t slot = (fpair) * p.maxseg + kslot;                            \
    float* dst = p.part[role] + slot * kTile * R + l;                           \
    _Pragma("unroll") for (int i = 0; i < RH; ++i) {                            \
      const int rr = 8 * (hq + 4 * i);                                          \
      _Pragma("unroll") for (int j = 0; j < 8; ++j) {                           \
        if (rr + j < R) dst[(rr + j) * kTile] = A[8 * i + j];                   \
        A[8 * i + j] = 0.f;                                                     \
      }                                                                         \
    }                                                                           \
  } while (0)
#ifdef KRP_DEV_TRACE
  long long sec_acc_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  KRP_SEC_BEGIN();
  for (int64_t t = t0; t < t1; ++t) {
    KRP_SEC(7);
    if (pair != prev_pair) {
      if (DOA && prev_pair >= 0) KRP_FLUSH(prev_pair);
      prev_pair = pair;
      const int rb = static_cast<int>(pair / CB), cb = static_cast<int>(pair - static_cast<int64_t>(rb) * CB);
      const int kblk = role == kRoleP ? cb : rb, mblk = role == kRoleP ? rb : cb;
      // B image of this segment (out of line: rare, and large once unrolled — it would crowd the hot loop
      // out of the instruction cache)
      gen_bimage(p, smem_u32(bimg), kg0, kg1, kgsize, kblk, R, R8, DN, ew, lane);
      fence_proxy_async_smem();
      named_bar_sync(1, kNumEpiWarps * 32);
      if (ew == 0 && lane == 0) mbar_arrive(kb.b_ready);
      if (ew == 0 && lane == 0) KRP_TRACE(11, t - t0);
      if (TT != 0 && t_warp) {  // this lane's own Khatri-Rao row (the other contraction's operand) for T
        const uint32_t lin = static_cast<uint32_t>(mblk) * kTile + static_cast<uint32_t>(l);
        const bool inb = lin < mgsize;
#pragma unroll
        for (int i = 0; i < RH; ++i) {
          float w8[8];
          kr_row<8>(p, mg0, mg1, lin, 8 * (hq + 4 * i), inb ? R : 0, w8);
#pragma unroll
          for (int j = 0; j < 8; ++j) W[8 * i + j] = w8[j];
        }
      }
    }
    // Ω_S(s, ·) of this tile into the warp's row (fetched one tile ahead), then the next tile's fetch
    if constexpr (DOA) {
      __syncwarp();  // the previous tile's reads of the row are done
      float o0, o1;
      if (one_slice) {
        o0 = om_nx.v[0][0];
        o1 = om_nx.v[0][1];
      } else {
        o0 = om_nx.x0, o1 = om_nx.x1;
#pragma unroll
        for (int q = 0; q < kOmsDefer; ++q) o0 *= om_nx.v[q][0], o1 *= om_nx.v[q][1];
        o0 = c0ok ? o0 : 0.f;
        o1 = c1ok ? o1 : 0.f;
      }
      oms_w[lane] = o0;
      oms_w[lane + 32] = o1;
      __syncwarp();
      if (t + 1 < t1) KRP_OMS_FETCH(s + 1 == S ? 0 : s + 1);
    }
    KRP_SEC(0);
    KWAIT(&kb.acc_full[ast], aph);
    KRP_SEC(1);
    tc_fence_after();
    const uint32_t tD = tacc + static_cast<uint32_t>(ast * DN);
    const uint32_t rbuf_s = rbuf0 + static_cast<uint32_t>(parity) * (4 * 64 * 4);
    // every round's accumulator columns are loaded before a single wait (TMEM reads queue behind the MMAs'
    // operand traffic, so one wait per tile instead of one per round)
    float za[RH][8], zb[RH][8];
#pragma unroll
    for (int i = 0; i < RH; ++i) {
      if (i < nval) {
        const uint32_t rr = static_cast<uint32_t>(8 * (hq + 4 * i));
        tmem_ld8(tD + rr, za[i]);
        tmem_ld8(tD + static_cast<uint32_t>(R8) + rr, zb[i]);
      }
    }
    tmem_ld_wait();
    KRP_SEC(2);
#pragma unroll
    for (int i = 0; i < RH; ++i) {
      if (i < nval) {
        const int rr = 8 * (hq + 4 * i);
        float z[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const float2 v = f2_add(make_float2(za[i][j], za[i][j + 1]), make_float2(zb[i][j], zb[i][j + 1]));
          z[j] = v.x;
          z[j + 1] = v.y;
        }
        if constexpr (DOA) {
          float om8[8];
          lds_v4(oms_s + rr * 4, om8[0], om8[1], om8[2], om8[3]);
          lds_v4(oms_s + rr * 4 + 16, om8[4], om8[5], om8[6], om8[7]);
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const float2 c = f2_fma(make_float2(z[j], z[j + 1]), make_float2(om8[j], om8[j + 1]),
                                    make_float2(A[8 * i + j], A[8 * i + j + 1]));
            A[8 * i + j] = c.x;
            A[8 * i + j + 1] = c.y;
          }
        }
        if (TT != 0 && t_warp) {
          float tv[8];
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const float2 tw = f2_mul(make_float2(z[j], z[j + 1]), make_float2(W[8 * i + j], W[8 * i + j + 1]));
            tv[j] = tw.x;
            tv[j + 1] = tw.y;
          }
          const float tsum = butterfly8(tv, lane);
          if ((lane & 3) == 0) sts_f32(rbuf_s + (rr + (lane >> 2)) * 4, tsum);
        }
      }
    }
    KRP_SEC(3);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&kb.acc_empty[ast]);
    if (++ast == kNA) {
      ast = 0;
      aph ^= 1;
    }
    if (TT != 0 && t_warp) {  // fixed-order sum of the four lane quarters for this role's T columns
      KRP_SEC(4);
      named_bar_sync(2, t_threads);
      KRP_SEC(5);
      // the T warps, renumbered 0..(t_threads/32 - 1), take one column each
      const int tw = TT == 3 ? static_cast<int>(ew) : (hq >> 1) * 4 + static_cast<int>(sub);
      const int e = tw * 32 + static_cast<int>(lane);
      const bool mine = TT == 3 || (TT == 1 && ((e >> 3) & 1) == 0) || (TT == 2 && ((e >> 3) & 1) == 1);
      if (e < R && mine) {
        const float* rb_ = red + parity * 4 * 64;
        const float tot = ((rb_[e] + rb_[64 + e]) + rb_[128 + e]) + rb_[192 + e];
        p.Tpart[(pair * S + s) * R + e] = tot;
      }
      parity ^= 1;
      KRP_SEC(6);
    }
    if (++s == S) {
      s = 0;
      ++pair;
    }
  }
  if (DOA && prev_pair >= 0) KRP_FLUSH(prev_pair);
#undef KRP_FLUSH
#undef KRP_OMS_FETCH
#ifdef KRP_DEV_TRACE
  if (p.trace && blockIdx.x < 2 && lane == 0 && ew < 8)
    for (int i = 0; i < 8; ++i) p.trace[(blockIdx.x * 16 + 14 + (ew >> 2)) * 64 + (ew & 3) * 8 + i] = sec_acc_[i];
#endif
}

template <int RH>
__global__ void __launch_bounds__(kThreads, 1)
    krp_tc_sketch_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 operands need 1 KB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.sm_bar);
  KBars kb;
  kb.full_x = bars;
  kb.empty_x = kb.full_x + p.NS;
  kb.chunk_full = kb.empty_x + p.NS;
  kb.chunk_ready = kb.chunk_full + 4;
  kb.acc_full = kb.chunk_ready + 4;
  kb.acc_empty = kb.acc_full + kNA;
  kb.b_ready = kb.acc_empty + kNA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kb.b_ready + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int rank = p.clustered ? static_cast<int>(cluster_ctarank()) : static_cast<int>(blockIdx.x & 1u);
  const int role = p.pairs ? rank : p.role_fixed;
  const int grp = p.pairs ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const bool q_ss = role == kRoleQ && !p.qhi_tmem;  // the Q MMA reads A_hi from the tile stage
  const int NC = p.NC[role];
  const int ccols = p.ccols[role];

  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x == 0) {
    // stage consumers: 8 split warps (+ the Q commit) of this CTA, and of the peer when the tile is multicast
    const uint32_t qss_any = p.qhi_tmem ? 0u : 1u;
    const uint32_t empty_count = p.clustered ? 2u * kNumSplitWarps + qss_any : kNumSplitWarps + (q_ss ? 1u : 0u);
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&kb.full_x[i], 1);
      mbar_init(&kb.empty_x[i], empty_count);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&kb.chunk_full[i], 4);
      mbar_init(&kb.chunk_ready[i], 1);
    }
    for (int i = 0; i < kNA; ++i) {
      mbar_init(&kb.acc_full[i], 1);
      mbar_init(&kb.acc_empty[i], kNumEpiWarps);
    }
    mbar_init(kb.b_ready, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  if (p.clustered) cluster_sync();  // the peer's barriers are initialised before any multicast / remote arrive
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  pdl_launch_dependents();  // the assembly kernel may be scheduled now (it waits for this grid to finish)

  const int ngrp = p.ncl;
  const int64_t t0 = static_cast<int64_t>(grp) * p.T / ngrp;
  const int64_t t1 = static_cast<int64_t>(grp + 1) * p.T / ngrp;

  if (warp >= kTmaWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsProd));
    if (warp == kTmaWarp) {
      // ------------------------------------------------------------ TMA producer
      if (elect_one()) {
        pdl_wait();  // X may be written by the previous kernel in the stream
        tma_prefetch_desc(&tmap);
        const uint64_t pol = policy_evict_first();
        // boxes this CTA issues: all four, or (multicast) two of them for both CTAs of the cluster
        const int jb = p.clustered ? rank : 0, js = p.clustered ? 2 : 1;
        int st = 0;
        uint32_t ph = 0;
        int64_t pair = t0 / p.S, s = t0 % p.S;
        int rb = static_cast<int>(pair / p.CB), cb = static_cast<int>(pair % p.CB);
        constexpr int kPf = KRP_PF_DIST;  // L2 prefetch distance (tiles)
        int64_t pf_t = t0, pf_pair = pair, pf_s = s;
#define KRP_PF_ISSUE()                                                                            \
  do {                                                                                            \
    const int pp = static_cast<int>(pf_pair), prb = pp / p.CB, pcb = pp - prb * p.CB;             \
    for (int j = jb; j < 4; j += js)                                                              \
      tma_prefetch_3d(&tmap, prb * kTile + 32 * j, pcb * kTile, static_cast<int32_t>(pf_s));      \
    if (++pf_s == p.S) {                                                                          \
      pf_s = 0;                                                                                   \
      ++pf_pair;                                                                                  \
    }                                                                                             \
    ++pf_t;                                                                                       \
  } while (0)
        for (int i = 0; i < kPf && pf_t < t1; ++i) KRP_PF_ISSUE();
        for (int64_t t = t0; t < t1; ++t) {
          if (pf_t < t1) KRP_PF_ISSUE();
          KRP_TRACE(0, t - t0);
          KWAIT(&kb.empty_x[st], ph ^ 1);
          KRP_TRACE(1, t - t0);
          mbar_arrive_expect_tx(&kb.full_x[st], kStageBytes);
          uint8_t* dst = smem + st * kStageBytes;
          for (int j = jb; j < 4; j += js) {
            if (p.clustered)
              tma_load_3d_mc(dst + j * 16384, &tmap, &kb.full_x[st], rb * kTile + 32 * j, cb * kTile,
                             static_cast<int32_t>(s), 0x3, pol);
            else
              tma_load_3d(dst + j * 16384, &tmap, &kb.full_x[st], rb * kTile + 32 * j, cb * kTile,
                          static_cast<int32_t>(s), pol);
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
#undef KRP_PF_ISSUE
      }
    } else if (warp == kMmaWarp) {
      // ------------------------------------------------------------ MMA issuer
      const bool leader = elect_one();
      const uint32_t idesc1 = make_idesc_tf32(128, p.DN, 0, 0);  // hi x [B_hi | B_lo]
      const uint32_t idesc2 = make_idesc_tf32(128, p.N2, 0, 0);  // lo x B_hi
      const uint64_t bdesc0 = make_smem_desc(smem_u32(smem + p.sm_b), 0, 1024, kLayoutSW128);
      const uint64_t adesc0 = make_smem_desc(smem_u32(smem), 0, 1024, kLayoutSW128);
      const uint64_t katom_d = static_cast<uint64_t>(p.DN) * 8;  // one 32-wide K atom of B: (DN*128 B) >> 4
      const uint32_t lo_off = (role == kRoleP || p.qhi_tmem) ? kCH : 0;  // lo columns inside a chunk slot
      int ast = 0, xst = 0, cst = 0;
      uint32_t aph = 0, bph = 0, cph = 0;
      int64_t s_cur = t0 % p.S;
      bool first = true;
      for (int64_t t = t0; t < t1; ++t) {
        if (first || s_cur == 0) {  // a new (ρ-block, γ-block) segment: wait for its B image
          KWAIT(kb.b_ready, bph);
          bph ^= 1;
          first = false;
        }
        MMA_WAIT(&kb.acc_empty[ast], aph ^ 1);
        if (leader) KRP_TRACE(2, t - t0);
        tc_fence_after();
        const uint32_t dA = tbase + p.tm_acc + ast * p.DN;
        const uint64_t adesc_t = adesc0 + ((static_cast<uint64_t>(xst) * kStageBytes) >> 4);
        for (int kc = 0; kc < kNkc; ++kc) {
          MMA_WAIT(&kb.chunk_full[cst], cph);
          tc_fence_after();
          const uint32_t ach = tbase + p.tm_chunk + cst * ccols;
          if (leader) {
#pragma unroll
            for (int ks = 0; ks < kCH / 8; ++ks) {
              const int kk = kc * (kCH / 8) + ks;
              const uint32_t acc0 = kk > 0 ? 1u : 0u;
              const uint64_t bd = bdesc0 + static_cast<uint64_t>(kk >> 2) * katom_d + (kk & 3) * 2;
              if (q_ss)  // A_hi: the raw tile, box kk/4 (16 KB), K offset (kk & 3) * 32 B
                mma_tf32_ss(dA, adesc_t + static_cast<uint64_t>(kk >> 2) * 1024 + (kk & 3) * 2, bd, idesc1, acc0);
              else
                mma_tf32_ts(dA, ach + 8 * ks, bd, idesc1, acc0);
              mma_tf32_ts(dA, ach + lo_off + 8 * ks, bd, idesc2, 1u);
            }
            mma_commit(&kb.chunk_ready[cst]);
          }
          __syncwarp();
          if (++cst == NC) {
            cst = 0;
            cph ^= 1;
          }
        }
        if (leader) {
          if (q_ss) {  // the raw tile may be overwritten once these MMAs finish
            if (p.clustered) mma_commit_mc(&kb.empty_x[xst], 0x3);
            else mma_commit(&kb.empty_x[xst]);
          }
          mma_commit(&kb.acc_full[ast]);
          KRP_TRACE(3, t - t0);
        }
        __syncwarp();
        if (++xst == p.NS) xst = 0;
        if (++ast == kNA) {
          ast = 0;
          aph ^= 1;
        }
        if (++s_cur == p.S) s_cur = 0;
      }
    }
  } else if (warp < kNumSplitWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsSplit));
    const int ntile = static_cast<int>(t1 - t0);
    const uint32_t smem0 = smem_u32(smem);
    if (role == kRoleP) split_loop<kRoleP, false>(p, kb, smem0, tbase, ntile, NC, ccols, rank, warp, lane);
    else if (p.qhi_tmem) split_loop<kRoleQ, true>(p, kb, smem0, tbase, ntile, NC, ccols, rank, warp, lane);
    else split_loop<kRoleQ, false>(p, kb, smem0, tbase, ntile, NC, ccols, rank, warp, lane);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
    pdl_wait();  // reads the Ω_k, overwrites partial slots the previous assembly kernel may still read
    const bool do_a = p.do_a[role] != 0;
    // T: on one role it does every round; a pair splits it (P the even, Q the odd i of each thread)
    const int tt = p.t_role == role ? 3 : (p.t_role == kTBoth ? (role == kRoleP ? 1 : 2) : 0);
    if (do_a) {
      switch (tt) {
        case 0: epi_loop<RH, true, 0>(p, kb, smem, tbase, role, grp, t0, t1, warp, lane); break;
        case 1: epi_loop<RH, true, 1>(p, kb, smem, tbase, role, grp, t0, t1, warp, lane); break;
        case 2: epi_loop<RH, true, 2>(p, kb, smem, tbase, role, grp, t0, t1, warp, lane); break;
        default: epi_loop<RH, true, 3>(p, kb, smem, tbase, role, grp, t0, t1, warp, lane); break;
      }
    } else {
      epi_loop<RH, false, 3>(p, kb, smem, tbase, role, grp, t0, t1, warp, lane);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.clustered) cluster_sync();  // no remote arrive / multicast may target an exited CTA
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ reduction of partials + multi-TTVs
struct RedParams {
  int64_t M, C, S, T;
  int RB, CB, R, ngrp, maxseg, ldy;
  int do_p, do_q, do_t;
  const float *partA1, *partA2, *Tpart;
  float *Pm, *Qc, *Ts;
  float *outP, *outQ, *outT;  // non-null: the group is a single wanted mode, write its Y directly (row stride ldy)
};

// P(ρ,r) = Σ_{cb} Σ_{k < nk(pair)} partA1[(rb*CB + cb)*maxseg + k][r][ρ%128]
// Qc(γ,r) likewise over rb;  Ts(s,r) = Σ_{pairs} Tpart[pair][s][r].
// One block = 32 outputs x 8 warps: for P / Qc the 32 lanes take 32 consecutive rows ρ of one column r
// (coalesced partial reads), for Ts 32 consecutive (s, r).  The flattened term list is split into 8
// contiguous shares, each summed in order, then warp 0 adds the 8 shares in order: a fixed reduction tree
// (deterministic).  nk(pair) = the number of tile groups that touched the pair, from the static tile split.
constexpr int kRedWarps = 8;
constexpr int kAsmMaxOther = 1024;
__global__ void __launch_bounds__(256) tc_assemble_kernel(const __grid_constant__ RedParams p) {
  __shared__ float red[kRedWarps][32];
  __shared__ int s_pnk[kAsmMaxOther];
  const int w = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  const int64_t nP = p.do_p ? p.M * p.R : 0, nQ = p.do_q ? p.C * p.R : 0, nT = p.do_t ? p.S * p.R : 0;
  const int64_t bP = p.do_p ? (p.M + 31) / 32 * p.R : 0, bQ = p.do_q ? (p.C + 31) / 32 * p.R : 0;
  int64_t blk_id = blockIdx.x;
  int region;
  if (blk_id < bP) {
    region = 0;
  } else if ((blk_id -= bP) < bQ) {
    region = 1;
  } else {
    blk_id -= bQ;
    region = 2;
  }
  int64_t idx = blk_id * 32 + lane;
  bool valid = true;
  float acc = 0.f;
  int outr = 0;
  int64_t outi = 0;
  if (region < 2) {
    const bool rows = region == 0;
    const int64_t nrow = rows ? p.M : p.C;
    const int r = static_cast<int>(blk_id % p.R);
    const int64_t rho = (blk_id / p.R) * 32 + lane;
    valid = rho < nrow;
    const int64_t rc = valid ? rho : nrow - 1;
    idx = rc * p.R + r;
    outi = rc;
    outr = r;
    const int blk = static_cast<int>(rc / kTile), l = static_cast<int>(rc % kTile);
    const float* part = (rows ? p.partA1 : p.partA2) + static_cast<int64_t>(r) * kTile + l;
    const int64_t kstride = static_cast<int64_t>(kTile) * p.R;
    const int nother = rows ? p.CB : p.RB;
    const bool spnk = nother <= kAsmMaxOther;
    auto pnk = [&](int o) {
      const int64_t pr = rows ? (static_cast<int64_t>(blk) * p.CB + o) : (static_cast<int64_t>(o) * p.CB + blk);
      return grp_of_tile((pr + 1) * p.S - 1, p.T, p.ngrp) - grp_of_tile(pr * p.S, p.T, p.ngrp) + 1;
    };
    if (spnk)
      for (int o = static_cast<int>(threadIdx.x); o < nother; o += blockDim.x) s_pnk[o] = pnk(o);
    __syncthreads();
    pdl_wait();  // the partials are written by the sketch kernel
    const int64_t F = static_cast<int64_t>(nother) * p.maxseg;  // flattened (other block, slot) terms
    const int64_t f0 = w * F / kRedWarps, f1 = (w + 1) * F / kRedWarps;
    for (int64_t f = f0; f < f1; f += 8) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = 0.f;
        const int64_t ff = f + i;
        if (ff < f1) {
          const uint32_t f32 = static_cast<uint32_t>(ff), o = f32 / static_cast<uint32_t>(p.maxseg);
          const uint32_t k = f32 - o * static_cast<uint32_t>(p.maxseg);
          const int64_t pair = rows ? (static_cast<int64_t>(blk) * p.CB + o) : (static_cast<int64_t>(o) * p.CB + blk);
          const int nk = spnk ? s_pnk[o] : pnk(static_cast<int>(o));
          if (static_cast<int>(k) < nk) v[i] = __ldg(part + (pair * p.maxseg + k) * kstride);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += v[i];
    }
  } else {
    pdl_wait();  // Tpart is written by the sketch kernel
    const uint32_t idc = static_cast<uint32_t>(idx < nT ? idx : nT - 1);
    const uint32_t s = idc / static_cast<uint32_t>(p.R);
    const int r = static_cast<int>(idc - s * static_cast<uint32_t>(p.R));
    outi = s;
    outr = r;
    const int64_t npairs = static_cast<int64_t>(p.RB) * p.CB;
    const int64_t p0 = w * npairs / kRedWarps, p1 = (w + 1) * npairs / kRedWarps;
    const int64_t pstride = p.S * p.R;
    const float* src = p.Tpart + static_cast<int64_t>(s) * p.R + r;
    for (int64_t q = p0; q < p1; q += 8) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = (q + i < p1) ? __ldg(src + (q + i) * pstride) : 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += v[i];
    }
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    float tot = red[0][lane];
#pragma unroll
    for (int i = 1; i < kRedWarps; ++i) tot += red[i][lane];
    const int64_t n = region == 0 ? nP : (region == 1 ? nQ : nT);
    if (valid && idx < n) {
      float* direct = region == 0 ? p.outP : (region == 1 ? p.outQ : p.outT);
      if (direct) direct[outi * p.ldy + outr] = tot;
      else (region == 0 ? p.Pm : (region == 1 ? p.Qc : p.Ts))[idx] = tot;
    }
  }
}

int64_t assemble_blocks(int64_t M, int64_t C, int64_t S, int R, int do_p, int do_q, int do_t) {
  return (do_p ? (M + 31) / 32 * R : 0) + (do_q ? (C + 31) / 32 * R : 0) + (do_t ? (S * R + 31) / 32 : 0);
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

// ------------------------------------------------------------------ input staging for shapes TMA cannot view
// Xp(ρ, γs) = X(ρ, γs) for ρ < M, 0 for M <= ρ < Mp (Mp = round4(M): 16-byte row pitch), also used for a
// base address that is not 16-byte aligned.  One extra pass over X; only for such shapes.
__global__ void repack_rows_kernel(const float* __restrict__ X, int64_t M, int64_t Mp, int64_t cols,
                                   float* __restrict__ Xp) {
  const int64_t total = Mp * cols;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / Mp, r = e - c * Mp;
    Xp[e] = r < M ? X[c * M + r] : 0.f;
  }
}

// ------------------------------------------------------------------ host planning
struct TcPlan {
  bool ok = false;
  int m = 0, m2 = 0;
  int64_t M = 0, Mp = 0, C = 0, S = 0;
  int RB = 0, CB = 0;
  int64_t T = 0;
  int R = 0, R8 = 0, N2 = 0, DN = 0, NS = 0, RH = 0;
  int NC[2] = {0, 0}, ccols[2] = {0, 0};
  int pairs = 0, clustered = 0, role_fixed = 0, t_role = -1, qhi_tmem = 0;
  int do_a[2] = {0, 0};
  int do_p = 0, do_q = 0, do_t = 0;  // which group objects exist (A1, A2, T)
  int grid = 0, ncl = 0, maxseg = 0, nslot = 0;
  int tm_acc = 0, tm_chunk = 0;
  uint32_t sm_b = 0, sm_red = 0, sm_oms = 0, sm_bar = 0, smem_bytes = 0;
  bool repack = false;
  double cost = 0;
};

struct DevInfo {
  int sms = 148;
  bool sm100 = false;
  int max_clusters = -1;  // co-resident 2-CTA clusters of the sketch kernel (queried once per device)
};
DevInfo& dev_info() {
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

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Fill geometry for a grouping (m, m2) and check the kernel's constraints.
bool fill_plan(const Dims& g, int R, int m, int m2, const bool* want, bool allow_repack, TcPlan& pl) {
  pl = TcPlan{};
  int64_t M = 1, C = 1, S = 1;
  for (int k = 0; k < m; ++k) M *= g.n[k];
  for (int k = m; k < m2; ++k) C *= g.n[k];
  for (int k = m2; k < g.d; ++k) S *= g.n[k];
  const bool need_repack = (M % 4) != 0;
  if (need_repack && !allow_repack) return false;
  const int64_t Mp = (M + 3) / 4 * 4;
  // 32-bit index math in the kernels (group indices, partial offsets) and TMA coordinate limits
  if (Mp >= (int64_t(1) << 31) || C >= (int64_t(1) << 31) || S >= (int64_t(1) << 31)) return false;
  if (Mp * 64 >= (int64_t(1) << 31) || C * 64 >= (int64_t(1) << 31) || S * 64 >= (int64_t(1) << 31)) return false;
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
  pl.Mp = Mp;
  pl.C = C;
  pl.S = S;
  pl.repack = need_repack;
  pl.RB = static_cast<int>((Mp + kTile - 1) / kTile);
  pl.CB = static_cast<int>((C + kTile - 1) / kTile);
  pl.T = static_cast<int64_t>(pl.RB) * pl.CB * S;
  pl.R = R;
  pl.R8 = (R + 7) / 8 * 8;
  pl.N2 = (R + 15) / 16 * 16;
  pl.DN = 2 * pl.R8;
  pl.RH = (pl.R8 / 8 + 3) / 4;  // rounds per epilogue thread (16 warps: four per lane quarter)
  pl.qhi_tmem = env_int("KRP_TC_QHI_TMEM", 0) ? 1 : 0;
  // which role produces T: the side that is computed anyway; with both sides, KRP_TC_T_ROLE (default Q)
  int t_role = -1;
  if (ws) {
    if (wr && !wc) t_role = kRoleP;
    else if (wc && !wr) t_role = kRoleQ;
    else if (wr && wc) t_role = env_int("KRP_TC_T_ROLE", kTBoth);  // a pair: split T between its two roles
    else t_role = kRoleQ;                                           // slice modes only
  }
  pl.t_role = t_role;
  const bool needP = wr || t_role == kRoleP, needQ = wc || t_role == kRoleQ;
  pl.do_a[kRoleP] = wr ? 1 : 0;
  pl.do_a[kRoleQ] = wc ? 1 : 0;
  pl.do_p = wr ? 1 : 0;
  pl.do_q = wc ? 1 : 0;
  pl.do_t = ws ? 1 : 0;
  pl.pairs = needP && needQ ? 1 : 0;
  pl.role_fixed = needP ? kRoleP : kRoleQ;
  // TMEM (512 columns): 2 accumulator stages of DN, then chunk slots (P: hi + lo, Q: lo [+ hi])
  pl.tm_acc = 0;
  pl.tm_chunk = kNA * pl.DN;
  pl.ccols[kRoleP] = 2 * kCH;
  pl.ccols[kRoleQ] = pl.qhi_tmem ? 2 * kCH : kCH;
  for (int r = 0; r < 2; ++r) {
    pl.NC[r] = std::min(4, (512 - pl.tm_chunk) / pl.ccols[r]);
    if (pl.NC[r] < 2) return false;
  }
  // SMEM: NS tile stages (64 KB), the B image (DN rows x 512 B), T scratch, Ω_S rows, barriers
  const uint32_t bbytes = static_cast<uint32_t>(pl.DN) * 512u;
  const uint32_t misc = 2 * 4 * 64 * 4 + kNumEpiWarps * 64 * 4 + 256;
  const uint32_t cap = 232448;  // max dynamic shared memory per block (sm_100)
  const int ns = static_cast<int>((cap - bbytes - misc) / kStageBytes);
  if (ns < 1) return false;
  pl.NS = std::min(ns, 4);
  pl.sm_b = pl.NS * kStageBytes;
  pl.sm_red = pl.sm_b + bbytes;
  pl.sm_oms = pl.sm_red + 2 * 4 * 64 * 4;
  pl.sm_bar = pl.sm_oms + kNumEpiWarps * 64 * 4;
  pl.smem_bytes = pl.sm_bar + 256;
  // grid: one CTA per SM; pairs of CTAs (P, Q) when both sides are needed
  DevInfo& di = dev_info();
  const int sms = di.sms;
  const int want_cluster = env_int("KRP_TC_CLUSTER", 1);
  if (pl.pairs) {
    int ngrp = sms / 2;
    pl.clustered = want_cluster ? 1 : 0;
    if (pl.clustered && di.max_clusters > 0) ngrp = std::min(ngrp, di.max_clusters);
    ngrp = static_cast<int>(std::min<int64_t>(ngrp, pl.T));
    pl.ncl = ngrp;
    pl.grid = 2 * ngrp;
  } else {
    pl.ncl = static_cast<int>(std::min<int64_t>(sms, pl.T));
    pl.grid = pl.ncl;
  }
  // tile groups per (rb, cb) pair: a pair's S consecutive tiles meet at most ceil(S / floor(T/ncl)) + 1
  // consecutive groups of the static split
  {
    const int64_t per = std::max<int64_t>(1, pl.T / pl.ncl);
    pl.maxseg = static_cast<int>((S + per - 1) / per + 1);
    pl.nslot = static_cast<int>(static_cast<int64_t>(pl.RB) * pl.CB * pl.maxseg);
  }
  // cost in units of one tile pass of one role: per-SM tile work, per-segment overhead (B image, flush,
  // assembly ~8 tile passes per pair and role), and the repack pass
  const double roles = pl.pairs ? 2.0 : 1.0;
  const double pairs = static_cast<double>(pl.RB) * pl.CB;
  pl.cost = static_cast<double>(pl.T) * roles * (1.0 + 0.05 * pl.do_t) + 8.0 * pairs * roles +
            (need_repack ? 2.0 * static_cast<double>(g.N) / (kTile * kTile) : 0.0);
  pl.ok = true;
  return true;
}

bool choose_plan(const Dims& g, int R, const bool* want, bool force_repack, TcPlan& best) {
  if (R > kMaxTcR || R < 1) return false;
  bool found = false;
  for (int pass = 0; pass < 2 && !found; ++pass) {  // pass 1: groupings that need the repack
    const bool allow = pass == 1 || force_repack;
    for (int m = 1; m < g.d; ++m) {
      for (int m2 = m + 1; m2 <= g.d; ++m2) {
        TcPlan pl;
        if (!fill_plan(g, R, m, m2, want, allow, pl)) continue;
        if (force_repack) pl.repack = true;
        if (!found || pl.cost < best.cost) {
          best = pl;
          found = true;
        }
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

struct WsLayout {
  size_t a1, a2, tpart, pm, qc, ts, xp, total;
};
WsLayout ws_layout(const TcPlan& pl, const Dims& g) {
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
  w.tpart = take(pl.do_t ? static_cast<size_t>(pl.RB) * pl.CB * pl.S * pl.R * sizeof(float) : 0);
  w.pm = take(static_cast<size_t>(pl.M) * pl.R * sizeof(float));
  w.qc = take(static_cast<size_t>(pl.C) * pl.R * sizeof(float));
  w.ts = take(static_cast<size_t>(pl.S) * pl.R * sizeof(float));
  w.xp = take(pl.repack ? static_cast<size_t>(pl.Mp) * pl.C * pl.S * sizeof(float) : 0);
  (void)g;
  w.total = off;
  return w;
}

using KernFn = void (*)(const CUtensorMap, const TcParams);
KernFn kernel_for(int RH) {
  return RH <= 1 ? krp_tc_sketch_kernel<1> : krp_tc_sketch_kernel<2>;
}

// co-resident 2-CTA clusters of the sketch kernel at this shared-memory size (the persistent grid is sized to it)
int max_active_clusters(KernFn kern, uint32_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * dev_info().sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

// One launch sequence for R <= 64 columns: omega / Y pointers already offset to the column group,
// ldo / ldy = their row strides.
int tc_sketch_cols(const float* X, const Dims& g, const OmegaPtrs& om, int R, int ldo, const bool* want,
                   float* const* Y, int ldy, Arena& ar, cudaStream_t s) {
  const bool misaligned = (reinterpret_cast<uintptr_t>(X) & 15u) != 0;
  TcPlan pl;
  if (!choose_plan(g, R, want, misaligned, pl)) {
    set_error("tcgen05 sketch: no tiling for this shape");
    return KRP_EUNSUPPORTED;
  }
  auto encode = get_encode();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return KRP_EUNSUPPORTED;
  }
  const KernFn kern = kernel_for(pl.RH);
  KRP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(pl.smem_bytes)));
  if (pl.pairs && pl.clustered) {  // size the persistent grid to the co-resident clusters
    DevInfo& di = dev_info();
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    const int mc = max_active_clusters(kern, pl.smem_bytes);
    if (mc > 0 && mc < pl.ncl) {
      pl.ncl = mc;
      pl.grid = 2 * mc;
      const int64_t per = std::max<int64_t>(1, pl.T / pl.ncl);
      pl.maxseg = static_cast<int>((pl.S + per - 1) / per + 1);
      pl.nslot = static_cast<int>(static_cast<int64_t>(pl.RB) * pl.CB * pl.maxseg);
    }
    if (mc > 0) di.max_clusters = mc;
  }
  if (env_int("KRP_TC_VERBOSE", 0))
    fprintf(stderr,
            "[krp tc] dims M=%lld C=%lld S=%lld (m=%d m2=%d) RB=%d CB=%d T=%lld R=%d DN=%d NS=%d NC=%d/%d pairs=%d "
            "clustered=%d role=%d t_role=%d qhi_tmem=%d ncl=%d grid=%d maxseg=%d smem=%u repack=%d\n",
            (long long)pl.M, (long long)pl.C, (long long)pl.S, pl.m, pl.m2, pl.RB, pl.CB, (long long)pl.T, R, pl.DN,
            pl.NS, pl.NC[0], pl.NC[1], pl.pairs, pl.clustered, pl.role_fixed, pl.t_role, pl.qhi_tmem, pl.ncl,
            pl.grid, pl.maxseg, pl.smem_bytes, pl.repack ? 1 : 0);
  const WsLayout wl = ws_layout(pl, g);
  const size_t mark = ar.off;
  char* wsb = ar.take<char>(wl.total);
  if (ar.overflow()) {
    set_error("workspace too small for the tcgen05 sketch");
    return KRP_ENOMEM;
  }
  const float* Xv = X;
  if (pl.repack) {
    float* Xp = reinterpret_cast<float*>(wsb + wl.xp);
    const int64_t total = pl.Mp * pl.C * pl.S;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
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
  p.R8 = pl.R8;
  p.N2 = pl.N2;
  p.DN = pl.DN;
  p.ldo = ldo;
  p.NS = pl.NS;
  for (int r = 0; r < 2; ++r) {
    p.NC[r] = pl.NC[r];
    p.ccols[r] = pl.ccols[r];
    p.do_a[r] = pl.do_a[r];
  }
  p.pairs = pl.pairs;
  p.clustered = pl.clustered;
  p.role_fixed = pl.role_fixed;
  p.t_role = pl.t_role;
  p.qhi_tmem = pl.qhi_tmem;
  p.ncl = pl.ncl;
  p.maxseg = pl.maxseg;
  p.tm_acc = pl.tm_acc;
  p.tm_chunk = pl.tm_chunk;
  p.sm_b = pl.sm_b;
  p.sm_red = pl.sm_red;
  p.sm_oms = pl.sm_oms;
  p.sm_bar = pl.sm_bar;
  p.part[kRoleP] = reinterpret_cast<float*>(wsb + wl.a1);
  p.part[kRoleQ] = reinterpret_cast<float*>(wsb + wl.a2);
  p.Tpart = reinterpret_cast<float*>(wsb + wl.tpart);
  p.d = g.d;
  p.m = pl.m;
  p.m2 = pl.m2;
  int64_t gs[kMaxD];  // stride of mode k inside its group (rows / cols / slices)
  {
    int64_t st = 1;
    for (int k = 0; k < pl.m; ++k) gs[k] = st, st *= g.n[k];
    st = 1;
    for (int k = pl.m; k < pl.m2; ++k) gs[k] = st, st *= g.n[k];
    st = 1;
    for (int k = pl.m2; k < g.d; ++k) gs[k] = st, st *= g.n[k];
  }
  for (int k = 0; k < g.d; ++k) {
    p.n[k] = g.n[k];
    p.gs[k] = gs[k];
    p.om[k] = om.p[k];
  }
  p.trace = nullptr;
#ifdef KRP_DEV_TRACE
  static long long* trace_buf = nullptr;
  if (getenv("KRP_TC_TRACE")) {
    if (!trace_buf) cudaMalloc(&trace_buf, 2 * 16 * 64 * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0, 2 * 16 * 64 * sizeof(long long), s);
    p.trace = trace_buf;
  }
#endif
  float* Pm = reinterpret_cast<float*>(wsb + wl.pm);
  float* Qc = reinterpret_cast<float*>(wsb + wl.qc);
  float* Ts = reinterpret_cast<float*>(wsb + wl.ts);

  CUtensorMap tmap;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(pl.Mp), static_cast<cuuint64_t>(pl.C), static_cast<cuuint64_t>(pl.S)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(pl.Mp) * 4, static_cast<cuuint64_t>(pl.Mp * pl.C) * 4};
    cuuint32_t box[3] = {32, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(Xv), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d) for %lld x %lld x %lld", static_cast<int>(r),
                static_cast<long long>(pl.Mp), static_cast<long long>(pl.C), static_cast<long long>(pl.S));
      return KRP_ECUDA;
    }
  }
  // 1. the fused tile kernel (persistent; CTA pairs as 2-CTA clusters when both sides are needed)
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(pl.grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pl.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (pl.pairs && pl.clustered) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = 2;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    prof_begin(s);
    KRP_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, tmap, p));
    KRP_CHECK_LAUNCH();
    int nw = 0;
    for (int k = 0; k < g.d; ++k) nw += want[k] ? 1 : 0;
    // algorithmic work of this launch: X read once; 2*N*R flops per wanted side (4NR for all modes)
    const double sides = (pl.do_p || pl.do_q) && pl.do_t ? 2.0 : static_cast<double>((pl.do_p + pl.do_q) ? pl.do_p + pl.do_q : 1);
    prof_end(s, 4.0 * static_cast<double>(g.N), 2.0 * static_cast<double>(g.N) * R * (nw == g.d ? 2.0 : sides));
#ifdef KRP_DEV_TRACE
    if (p.trace) {
      static long long h[2 * 16 * 64];
      cudaMemcpyAsync(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (FILE* f = fopen(getenv("KRP_TC_TRACE"), "w")) {
        for (int i = 0; i < 2 * 16 * 64; ++i) fprintf(f, "%lld%c", h[i], (i % 64 == 63) ? '\n' : ' ');
        fclose(f);
      }
    }
#endif
  }
  // 2. fixed-order sum of the per-group partials, then the multi-TTVs of groups with several modes
  {
    RedParams rp{};
    rp.M = pl.M;
    rp.C = pl.C;
    rp.S = pl.S;
    rp.T = pl.T;
    rp.RB = pl.RB;
    rp.CB = pl.CB;
    rp.R = R;
    rp.ngrp = pl.ncl;
    rp.maxseg = pl.maxseg;
    rp.ldy = ldy;
    rp.do_p = pl.do_p;
    rp.do_q = pl.do_q;
    rp.do_t = pl.do_t;
    rp.partA1 = p.part[kRoleP];
    rp.partA2 = p.part[kRoleQ];
    rp.Tpart = p.Tpart;
    rp.Pm = Pm;
    rp.Qc = Qc;
    rp.Ts = Ts;
    rp.outP = (pl.m == 1 && want[0]) ? Y[0] : nullptr;
    rp.outQ = (pl.m2 - pl.m == 1 && want[pl.m]) ? Y[pl.m] : nullptr;
    rp.outT = (g.d - pl.m2 == 1 && want[pl.m2]) ? Y[pl.m2] : nullptr;
    if (rp.do_t && pl.RB * pl.CB == 1 && !rp.outT) {
      // one (ρ-block, γ-block) pair: the per-tile T rows already are Ts ([s][r]), read in place by the TTV
      Ts = p.Tpart;
      rp.do_t = 0;
    }
    const int64_t nblk = assemble_blocks(pl.M, pl.C, pl.S, R, rp.do_p, rp.do_q, rp.do_t);
    if (nblk > 0) {
      KRP_CHECK_CUDA(launch_pdl(tc_assemble_kernel, dim3(static_cast<unsigned>(nblk)), dim3(256), 0, s, rp));
      KRP_CHECK_LAUNCH();
    }
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

bool tc_device_ok() { return dev_info().sm100 && get_encode() != nullptr; }

size_t tc_sketch_ws_bytes(const Dims& g, int R, const bool* want) {
  size_t b = 0;
  for (int c0 = 0; c0 < R; c0 += kMaxTcR) {
    const int Rc = std::min(kMaxTcR, R - c0);
    for (int rep = 0; rep < 2; ++rep) {  // with and without the repack (alignment is known only at call time)
      TcPlan pl;
      if (choose_plan(g, Rc, want, rep == 1, pl)) b = std::max(b, ws_layout(pl, g).total);
    }
  }
  return b;
}

// Columns of a KRP sketch are independent (Lemma 2.3): R > 64 runs as column groups of <= 64
// (one pass over X each), with Ω / Y addressed through their row strides.
int tc_sketch(const float* X, const Dims& g, const OmegaPtrs& om, int R, const bool* want, float* const* Y, Arena& ar,
              cudaStream_t s) {
  if (!tc_device_ok()) {
    set_error("the KRP sketch needs an sm_100a device (B200) and the CUDA driver's TMA encoder");
    return KRP_EUNSUPPORTED;
  }
  for (int c0 = 0; c0 < R; c0 += kMaxTcR) {
    const int Rc = std::min(kMaxTcR, R - c0);
    OmegaPtrs oc{};
    float* Yc[kMaxD] = {};
    for (int k = 0; k < g.d; ++k) {
      oc.p[k] = om.p[k] ? om.p[k] + c0 : nullptr;
      Yc[k] = (want[k] && Y[k]) ? Y[k] + c0 : nullptr;
    }
    KRP_TRY(tc_sketch_cols(X, g, oc, Rc, R, want, Yc, R, ar, s));
  }
  return KRP_OK;
}

}  // namespace krp
