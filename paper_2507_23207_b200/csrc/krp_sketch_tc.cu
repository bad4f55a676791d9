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
// Warp roles (448 threads): 0-3 split (TMEM lane quarters 0-3), 4-11 epilogue (two r-halves
// per lane quarter), 12 TMA producer, 13 MMA issuer.
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

constexpr int kThreads = 448;
constexpr int kEpiWarp0 = 4;
constexpr int kNumEpiWarps = 8;
constexpr int kTmaWarp = 12;
constexpr int kMmaWarp = 13;
constexpr int kCH = 16;             // TMEM A-chunk width (K columns per staged operand copy)
constexpr int kTile = 128;
constexpr int kStageFloats = 4 * 128 * 32;  // one 128x128 fp32 tile = 4 TMA boxes of {32, 128}
constexpr int kMaxTcR = 64;

struct TcParams {
  int64_t M, C, S;
  int RB, CB;
  int64_t T;
  int R, NP, N2;
  int NS, NC, NA;
  int do_p, do_q, do_t;
  int maxseg;
  int tm_acc, tm_chunk;
  uint32_t sm_x, sm_bp, sm_bq, sm_red, sm_bar;
  int m, m2, d;
  int64_t n[kMaxD];
  int64_t gs[kMaxD];  // stride of mode k inside its group (rows / cols / slices)
  const float* om[kMaxD];
  float* partA1;  // [nslot][128][R]
  float* partA2;
  int* slot_pair;  // [nslot]
  float* Tpart;    // [RB*CB][S][R]
  const float* WL;   // [M][R]  Khatri-Rao rows of the row modes
  const float* WR;   // [C][R]  Khatri-Rao rows of the col modes
  const float* OmS;  // [S][R]  Khatri-Rao rows of the slice modes
  int dbg;           // development bottleneck probes (KRP_TC_DEBUG): 0 normal, 1 TMA only,
                     // 2 TMA + split, 3 TMA + split + MMA (no epilogue)
};

__device__ __forceinline__ float omega_prod(const TcParams& p, int k0, int k1, int64_t lin, int r) {
  // Π_{k in [k0,k1)} Ω_k(i_k(lin), r), lin = linear index inside that mode group
  float w = 1.f;
  for (int k = k0; k < k1; ++k) {
    const int64_t ik = (lin / p.gs[k]) % p.n[k];
    w *= __ldg(p.om[k] + ik * p.R + r);
  }
  return w;
}

__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

template <int RMAX>
__global__ void __launch_bounds__(kThreads, 1)
    krp_tc_sketch_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xs = reinterpret_cast<float*>(smem + p.sm_x);
  uint8_t* bp = smem + p.sm_bp;
  uint8_t* bq = smem + p.sm_bq;
  float* red = reinterpret_cast<float*>(smem + p.sm_red);  // [2][4 lane quarters][RMAX]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.sm_bar);
  uint64_t* full_x = bars;
  uint64_t* empty_x = full_x + p.NS;
  uint64_t* chunk_full = empty_x + p.NS;
  uint64_t* chunk_empty = chunk_full + p.NC;
  uint64_t* acc_full = chunk_empty + p.NC;
  uint64_t* acc_empty = acc_full + p.NA;
  uint64_t* b_ready = acc_empty + p.NA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_ready + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&full_x[i], 1);
      mbar_init(&empty_x[i], 4);
    }
    for (int i = 0; i < p.NC; ++i) {
      mbar_init(&chunk_full[i], 4);
      mbar_init(&chunk_empty[i], 1);
    }
    for (int i = 0; i < p.NA; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kNumEpiWarps);
    }
    mbar_init(b_ready, 1);
    fence_barrier_init();
  }
  {  // zero both B operands once: rows >= 2R stay zero (UMMA N padding)
    float* b = reinterpret_cast<float*>(bp);
    const int nf = 2 * p.NP * 128;
    for (int i = threadIdx.x; i < nf; i += kThreads) b[i] = 0.f;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * p.T / gridDim.x;
  const int64_t t1 = static_cast<int64_t>(blockIdx.x + 1) * p.T / gridDim.x;
  const int nkc = kTile / kCH;

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmap);
      const uint64_t pol = policy_evict_first();
      int st = 0;
      uint32_t ph = 0;
      for (int64_t t = t0; t < t1; ++t) {
        const int64_t pair = t / p.S, s = t % p.S;
        const int rb = static_cast<int>(pair / p.CB), cb = static_cast<int>(pair % p.CB);
        if (p.dbg == 4) {  // probe: the producer consumes its own stages (no handshake)
          if (t - t0 >= p.NS) mbar_wait(&full_x[st], ph ^ 1);
        } else {
          mbar_wait(&empty_x[st], ph ^ 1);
        }
        mbar_arrive_expect_tx(&full_x[st], kStageFloats * 4);
        float* dst = xs + st * kStageFloats;
        for (int j = 0; j < 4; ++j)
          tma_load_3d(dst + j * 4096, &tmap, &full_x[st], rb * kTile + 32 * j, cb * kTile, static_cast<int32_t>(s),
                      pol);
        if (++st == p.NS) {
          st = 0;
          ph ^= 1;
        }
      }
      if (p.dbg == 4) {  // drain the stages still in flight
        for (int64_t t = std::max(t0, t1 - p.NS); t < t1; ++t) {
          const int s2 = static_cast<int>((t - t0) % p.NS);
          mbar_wait(&full_x[s2], static_cast<uint32_t>(((t - t0) / p.NS) & 1));
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (one thread)
    if (elect_one()) {
      const uint32_t idesc1 = make_idesc_tf32(128, p.NP, 0, 0);
      const uint32_t idesc2 = make_idesc_tf32(128, p.N2, 0, 0);
      const uint32_t bp_addr = smem_u32(bp), bq_addr = smem_u32(bq);
      int cst = 0, ast = 0;
      uint32_t cph = 0, aph = 0, bph = 0;
      int64_t prev_pair = -1;
      for (int64_t t = t0; t < ((p.dbg == 1 || p.dbg == 4) ? t0 : t1); ++t) {
        const int64_t pair = t / p.S;
        if (pair != prev_pair) {
          mbar_wait(b_ready, bph);
          bph ^= 1;
          prev_pair = pair;
        }
        if (p.dbg == 0) mbar_wait(&acc_empty[ast], aph ^ 1);
        tc_fence_after();
        const uint32_t dP = tbase + p.tm_acc + ast * 2 * p.NP;
        const uint32_t dQ = dP + p.NP;
        for (int kc = 0; kc < nkc; ++kc) {
          mbar_wait(&chunk_full[cst], cph);
          tc_fence_after();
          const uint32_t ch = tbase + p.tm_chunk + cst * 4 * kCH;
#pragma unroll
          for (int ks = 0; ks < kCH / 8; ++ks) {
            const int kk = kc * (kCH / 8) + ks;
            const uint32_t boff = (kk >> 2) * (p.NP * 128) + (kk & 3) * 32;
            if (p.dbg == 2) continue;
            if (p.do_p) {
              const uint64_t bd = make_smem_desc(bp_addr + boff, 0, 1024, kLayoutSW128);
              mma_tf32_ts(dP, ch + 0 * kCH + 8 * ks, bd, idesc1, kk > 0 ? 1u : 0u);  // hi x [B_hi | B_lo]
              mma_tf32_ts(dP, ch + 1 * kCH + 8 * ks, bd, idesc2, 1u);                 // lo x B_hi
            }
            if (p.do_q) {
              const uint64_t bd = make_smem_desc(bq_addr + boff, 0, 1024, kLayoutSW128);
              mma_tf32_ts(dQ, ch + 2 * kCH + 8 * ks, bd, idesc1, kk > 0 ? 1u : 0u);
              mma_tf32_ts(dQ, ch + 3 * kCH + 8 * ks, bd, idesc2, 1u);
            }
          }
          mma_commit(&chunk_empty[cst]);
          if (++cst == p.NC) {
            cst = 0;
            cph ^= 1;
          }
        }
        mma_commit(&acc_full[ast]);
        if (++ast == p.NA) {
          ast = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ split warps: SMEM tile -> TMEM hi/lo
    const uint32_t sub = warp;  // TMEM lane quarter
    const uint32_t lane_off = (32u * sub) << 16;
    int xst = 0, cst = 0;
    uint32_t xph = 0, cph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      mbar_wait(&full_x[xst], xph);
      const float* X = xs + xst * kStageFloats;
      if (p.dbg == 4) break;
      for (int kc = 0; kc < (p.dbg == 1 ? 0 : nkc); ++kc) {
        mbar_wait(&chunk_empty[cst], cph ^ 1);
        tc_fence_after();
        const uint32_t ch = tbase + lane_off + p.tm_chunk + cst * 4 * kCH;
        if (p.do_p) {
          // lane = ρ = 32*sub + lane (box `sub`), columns γ = kc*16 + j (rows of the box)
          const float* box = X + sub * 4096;
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int g = kc * 16 + j;
            const float x = box[g * 32 + ((((lane >> 2) ^ (g & 7))) << 2) + (lane & 3)];
            hi[j] = __float_as_uint(x);
            lo[j] = __float_as_uint(x - __uint_as_float(tf32_hi_bits(x)));
          }
          tmem_st16(ch + 0 * kCH, hi);
          tmem_st16(ch + 1 * kCH, lo);
        }
        if (p.do_q) {
          // lane = γ = 32*sub + lane, columns ρ = kc*16 + j : 16 consecutive ρ of row γ of box (kc/2)
          const int g = 32 * sub + lane;
          const float* row = X + (kc >> 1) * 4096 + g * 32;
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int chunk = ((kc & 1) * 4 + qq) ^ (g & 7);
            const float4 v = *reinterpret_cast<const float4*>(row + chunk * 4);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              hi[qq * 4 + e] = __float_as_uint(vv[e]);
              lo[qq * 4 + e] = __float_as_uint(vv[e] - __uint_as_float(tf32_hi_bits(vv[e])));
            }
          }
          tmem_st16(ch + 2 * kCH, hi);
          tmem_st16(ch + 3 * kCH, lo);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&chunk_full[cst]);
        if (++cst == p.NC) {
          cst = 0;
          cph ^= 1;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_x[xst]);
      if (++xst == p.NS) {
        xst = 0;
        xph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    // warps 4-7: P side (z1 -> A1 += z1·Ω_S, T = Σ_lanes z1·W_L);  warps 8-11: Q side (A2 += z2·Ω_S)
    const uint32_t ew = warp - kEpiWarp0;  // 0..7
    const uint32_t sub = warp & 3;         // TMEM lane quarter
    const bool pside = ew < 4;
    const int l = static_cast<int>(32 * sub + lane);
    const uint32_t lane_off = (32u * sub) << 16;
    const uint32_t k32 = static_cast<uint32_t>(l) & 31u, katom = static_cast<uint32_t>(l) >> 5;
    const bool active = pside ? (p.do_p != 0) : (p.do_q != 0);
    float A[RMAX];
#pragma unroll
    for (int j = 0; j < RMAX; ++j) A[j] = 0.f;
    int ast = 0;
    uint32_t aph = 0;
    int64_t prev_pair = -1;
    int seg = -1;
    int parity = 0;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t pair = t / p.S, s = t % p.S;
      if (pair != prev_pair) {
        if (prev_pair >= 0)
        {  // flush the finished segment's accumulators into its partial slot
          const int64_t slot = static_cast<int64_t>(blockIdx.x) * p.maxseg + seg;
          if (threadIdx.x == kEpiWarp0 * 32) p.slot_pair[slot] = static_cast<int>(prev_pair);
          float* dst = (pside ? p.partA1 : p.partA2) + (slot * kTile + l) * p.R;
#pragma unroll
          for (int j = 0; j < RMAX; ++j) {
            if (active && j < p.R) dst[j] = A[j];
            A[j] = 0.f;
          }
        }
        ++seg;
        prev_pair = pair;
        const int64_t rb = pair / p.CB, cb = pair % p.CB;
        // Khatri-Rao rows of this segment -> B operands [hi | lo] (K-major, SWIZZLE_128B).
        // P-side warps write B_Q (row lanes, W_L), Q-side warps write B_P (col lanes, W_R).
        if (pside ? (p.do_q || p.do_t) : p.do_p) {
          const int64_t lin = pside ? rb * kTile + l : cb * kTile + l;
          const bool inb = lin < (pside ? p.M : p.C);
          const float* tab = (pside ? p.WL : p.WR) + lin * p.R;
          uint8_t* base = (pside ? bq : bp) + katom * (p.NP * 128);
          for (int r = 0; r < p.R; ++r) {
            const float w = inb ? __ldg(tab + r) : 0.f;
            const float whi = __uint_as_float(tf32_hi_bits(w));
            *reinterpret_cast<float*>(base + sw128_offset(r, k32)) = whi;
            *reinterpret_cast<float*>(base + sw128_offset(p.R + r, k32)) = w - whi;
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, kNumEpiWarps * 32);
        if (threadIdx.x == kEpiWarp0 * 32) mbar_arrive(b_ready);
      }
      if (p.dbg != 0) continue;
      mbar_wait(&acc_full[ast], aph);
      tc_fence_after();
      const uint32_t tD = tbase + lane_off + p.tm_acc + ast * 2 * p.NP + (pside ? 0 : p.NP);
      const float* oms = p.OmS + s * p.R;
      const uint8_t* wlbase = bq + katom * (p.NP * 128);
      float* rbuf = red + parity * (4 * RMAX);
      const bool dot = pside && p.do_t;
#pragma unroll
      for (int rnd = 0; rnd < RMAX / 16; ++rnd) {
        const int rr = 16 * rnd;
        float tv[16];
        if (active) {
          float a[16], b[16];
          tmem_ld16(tD + rr, a);
          tmem_ld16(tD + p.R + rr, b);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int r = rr + j;
            float z = 0.f, ws = 0.f, wl = 0.f;
            if (r < p.R) {
              z = a[j] + b[j];
              ws = __ldg(oms + r);
              if (dot)
                wl = *reinterpret_cast<const float*>(wlbase + sw128_offset(r, k32)) +
                     *reinterpret_cast<const float*>(wlbase + sw128_offset(p.R + r, k32));
            }
            A[rr + j] = fmaf(z, ws, A[rr + j]);
            tv[j] = z * wl;
          }
        }
        if (rnd == RMAX / 16 - 1) {
          // every TMEM read of this tile is done: hand the accumulator stage back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[ast]);
        }
        if (dot) {
          // transposed butterfly over the 32 lanes: lanes 2q, 2q+1 end with the sum for r = rr + q
#pragma unroll
          for (int lvl = 0; lvl < 4; ++lvl) {
            const int m = 16 >> lvl;
            const int h = 8 >> lvl;
            const bool upper = (lane & m) != 0;
#pragma unroll
            for (int j = 0; j < h; ++j) {
              const float send = upper ? tv[j] : tv[j + h];
              const float keep = upper ? tv[j + h] : tv[j];
              tv[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
            }
          }
          tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 1);
          if ((lane & 1) == 0) rbuf[sub * RMAX + rr + (lane >> 1)] = tv[0];
        }
      }
      if (++ast == p.NA) {
        ast = 0;
        aph ^= 1;
      }
      if (dot) {
        // fixed-order sum of the four lane quarters (P-side warps only)
        named_bar_sync(2, 4 * 32);
        const int e = static_cast<int>(sub * 32 + lane);
        if (e < p.R) {
          const float tot = ((rbuf[e] + rbuf[RMAX + e]) + rbuf[2 * RMAX + e]) + rbuf[3 * RMAX + e];
          p.Tpart[(pair * p.S + s) * p.R + e] = tot;
        }
        parity ^= 1;
      }
    }
    if (prev_pair >= 0)
        {  // flush the finished segment's accumulators into its partial slot
          const int64_t slot = static_cast<int64_t>(blockIdx.x) * p.maxseg + seg;
          if (threadIdx.x == kEpiWarp0 * 32) p.slot_pair[slot] = static_cast<int>(prev_pair);
          float* dst = (pside ? p.partA1 : p.partA2) + (slot * kTile + l) * p.R;
#pragma unroll
          for (int j = 0; j < RMAX; ++j) {
            if (active && j < p.R) dst[j] = A[j];
            A[j] = 0.f;
          }
        }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ Khatri-Rao tables
struct TabParams {
  int d, m, m2, R;
  int64_t M, C, S;
  int64_t n[kMaxD];
  int64_t gs[kMaxD];
  const float* om[kMaxD];
  float *WL, *WR, *OmS;
};

// WL(ρ,r) = Π_{k<m} Ω_k(i_k(ρ),r), WR(γ,r) = Π_{m<=k<m2} Ω_k(..), OmS(s,r) = Π_{k>=m2} Ω_k(..)
__global__ void tc_tables_kernel(const __grid_constant__ TabParams p) {
  int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nl = p.M * p.R, nr = p.C * p.R, ns = p.S * p.R;
  int k0, k1;
  float* out;
  if (idx < nl) {
    k0 = 0, k1 = p.m, out = p.WL;
  } else if ((idx -= nl) < nr) {
    k0 = p.m, k1 = p.m2, out = p.WR;
  } else if ((idx -= nr) < ns) {
    k0 = p.m2, k1 = p.d, out = p.OmS;
  } else {
    return;
  }
  const int64_t lin = idx / p.R;
  const int r = static_cast<int>(idx - lin * p.R);
  float w = 1.f;
  for (int k = k0; k < k1; ++k) {
    const int64_t ik = (lin / p.gs[k]) % p.n[k];
    w *= __ldg(p.om[k] + ik * p.R + r);
  }
  out[idx] = w;
}

// ------------------------------------------------------------------ reduction of partials + multi-TTVs
struct RedParams {
  int64_t M, C, S, T;
  int RB, CB, R, grid, maxseg;
  int do_p, do_q, do_t;
  const float *partA1, *partA2, *Tpart;
  float *Pm, *Qc, *Ts;
};

// CTA owning tile t under the static split a0(b) = floor(b*T/grid)
__device__ __forceinline__ int cta_of(int64_t t, int64_t T, int grid) {
  return static_cast<int>(((t + 1) * grid - 1) / T);
}

// P(ρ,r) = Σ_{cb} Σ_{CTAs b of pair (rb,cb)} partA1[slot(b,pair)][ρ%128][r]   (fixed order)
// Qc(γ,r) likewise over rb;  Ts(s,r) = Σ_{pairs} Tpart[pair][s][r]
__global__ void tc_assemble_kernel(const __grid_constant__ RedParams p) {
  int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nP = p.do_p ? p.M * p.R : 0, nQ = p.do_q ? p.C * p.R : 0, nT = p.do_t ? p.S * p.R : 0;
  if (idx < nP + nQ) {
    const bool rows = idx < nP;
    if (!rows) idx -= nP;
    const int64_t lin = idx / p.R;
    const int r = static_cast<int>(idx - lin * p.R);
    const int blk = static_cast<int>(lin / kTile), l = static_cast<int>(lin % kTile);
    const float* part = rows ? p.partA1 : p.partA2;
    const int nother = rows ? p.CB : p.RB;
    float acc = 0.f;
    for (int o = 0; o < nother; ++o) {
      const int64_t pair = rows ? (static_cast<int64_t>(blk) * p.CB + o) : (static_cast<int64_t>(o) * p.CB + blk);
      const int b0 = cta_of(pair * p.S, p.T, p.grid), b1 = cta_of((pair + 1) * p.S - 1, p.T, p.grid);
      for (int b = b0; b <= b1; ++b) {
        const int64_t a0 = static_cast<int64_t>(b) * p.T / p.grid;
        const int64_t slot = static_cast<int64_t>(b) * p.maxseg + (pair - a0 / p.S);
        acc += part[(slot * kTile + l) * p.R + r];
      }
    }
    (rows ? p.Pm : p.Qc)[idx] = acc;
  } else if ((idx -= nP + nQ) < nT) {
    const int64_t s = idx / p.R;
    const int r = static_cast<int>(idx - s * p.R);
    const int64_t npairs = static_cast<int64_t>(p.RB) * p.CB;
    float acc = 0.f;
    for (int64_t pr = 0; pr < npairs; ++pr) acc += p.Tpart[(pr * p.S + s) * p.R + r];
    p.Ts[idx] = acc;
  }
}

struct TtvParams {
  int d, m, m2, R;
  int64_t M, C, S;
  int64_t n[kMaxD];
  int64_t gs[kMaxD];
  const float* om[kMaxD];
  const float *Pm, *Qc, *Ts;
  float* y[kMaxD];
  int want[kMaxD];
};

// Y_k(i, r) = Σ_{lin: i_k(lin) = i} src(lin, r) Π_{j in group, j != k} Ω_j(i_j(lin), r)
__global__ void tc_ttv_kernel(const __grid_constant__ TtvParams p) {
  int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int k = 0; k < p.d; ++k) {
    if (!p.want[k]) continue;
    const int64_t cnt = p.n[k] * p.R;
    if (idx >= cnt) {
      idx -= cnt;
      continue;
    }
    const int64_t i = idx / p.R;
    const int r = static_cast<int>(idx - i * p.R);
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
    double acc = 0.0;
    for (int64_t o = 0; o < others; ++o) {
      int64_t rem = o, lin = i * p.gs[k];
      float w = 1.f;
      for (int j = g0; j < g1; ++j) {
        if (j == k) continue;
        const int64_t ij = rem % p.n[j];
        rem /= p.n[j];
        lin += ij * p.gs[j];
        w *= __ldg(p.om[j] + ij * p.R + r);
      }
      acc += static_cast<double>(src[lin * p.R + r]) * w;
    }
    p.y[k][i * p.R + r] = static_cast<float>(acc);
    return;
  }
}

// ------------------------------------------------------------------ host planning
struct TcPlan {
  bool ok = false;
  int m = 0, m2 = 0;
  int64_t M = 0, C = 0, S = 0;
  int RB = 0, CB = 0;
  int64_t T = 0;
  int R = 0, NP = 0, N2 = 0, NS = 0, NC = 0, NA = 0;
  int do_p = 0, do_q = 0, do_t = 0;
  int grid = 0, maxseg = 0, nslot = 0;
  int tm_acc = 0, tm_chunk = 0;
  uint32_t sm_x = 0, sm_bp = 0, sm_bq = 0, sm_red = 0, sm_bar = 0, smem_bytes = 0;
};

int num_sms() {
  static int n = -1;
  if (n < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
                                                   cudaSuccess)
      n = 148;
  }
  return n;
}

bool device_is_sm100() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0, major = 0, minor = 0;
    ok = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess)
      ok = (major == 10 && minor == 0) ? 1 : 0;
    cudaGetLastError();
  }
  return ok == 1;
}

int round16(int v) { return (v + 15) / 16 * 16; }

// Fill geometry for a grouping (m, m2) and check the kernel's constraints.
bool fill_plan(const Dims& g, int R, int m, int m2, const bool* want, TcPlan& pl) {
  pl = TcPlan{};
  int64_t M = 1, C = 1, S = 1;
  for (int k = 0; k < m; ++k) M *= g.n[k];
  for (int k = m; k < m2; ++k) C *= g.n[k];
  for (int k = m2; k < g.d; ++k) S *= g.n[k];
  if (M < kTile || C < kTile || (M % 4) != 0) return false;
  if (M > (int64_t(1) << 31) || C > (int64_t(1) << 31) || S > (int64_t(1) << 31)) return false;
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
  pl.RB = static_cast<int>((M + kTile - 1) / kTile);
  pl.CB = static_cast<int>((C + kTile - 1) / kTile);
  pl.T = static_cast<int64_t>(pl.RB) * pl.CB * S;
  pl.R = R;
  pl.do_t = ws ? 1 : 0;
  pl.do_p = (wr || ws) ? 1 : 0;  // T is computed from z1
  pl.do_q = wc ? 1 : 0;
  pl.NP = round16(2 * R);
  pl.N2 = round16(R);
  // TMEM: NA accumulator stages of 2*NP columns, NC chunk stages of 4*kCH columns, 512 total
  pl.NA = (4 * pl.NP + 2 * 4 * kCH <= 512) ? 2 : 1;
  pl.NC = std::min(4, (512 - pl.NA * 2 * pl.NP) / (4 * kCH));
  if (pl.NC < 2) return false;
  pl.tm_acc = 0;
  pl.tm_chunk = pl.NA * 2 * pl.NP;
  // SMEM: X stages (64 KB each), B_P and B_Q (NP rows x 512 B each), reduction scratch, barriers
  const uint32_t bbytes = static_cast<uint32_t>(pl.NP) * 512u;
  const uint32_t misc = 2 * kNumEpiWarps * 32 * 4 + 512;
  const uint32_t budget = 232448 - 1024;
  int ns = static_cast<int>((budget - 2 * bbytes - misc) / (kStageFloats * 4));
  if (ns < 1) return false;
  pl.NS = std::min(ns, 3);
  pl.sm_x = 0;
  pl.sm_bp = pl.NS * kStageFloats * 4;
  pl.sm_bq = pl.sm_bp + bbytes;
  pl.sm_red = pl.sm_bq + bbytes;
  pl.sm_bar = pl.sm_red + 2 * kNumEpiWarps * 32 * 4;
  pl.smem_bytes = pl.sm_bar + 512 + 1024;
  pl.grid = static_cast<int>(std::min<int64_t>(num_sms(), pl.T));
  // segments per CTA (distinct (rb, cb) pairs in its contiguous tile range)
  int mx = 0;
  for (int b = 0; b < pl.grid; ++b) {
    const int64_t a0 = static_cast<int64_t>(b) * pl.T / pl.grid, a1 = static_cast<int64_t>(b + 1) * pl.T / pl.grid;
    if (a1 <= a0) continue;
    const int segs = static_cast<int>((a1 - 1) / S - a0 / S + 1);
    mx = std::max(mx, segs);
  }
  pl.maxseg = std::max(mx, 1);
  pl.nslot = pl.grid * pl.maxseg;
  pl.ok = true;
  return true;
}

bool choose_plan(const Dims& g, int R, const bool* want, TcPlan& best) {
  if (R > kMaxTcR || R < 1) return false;
  bool found = false;
  double best_cost = 1e300;
  for (int m = 1; m < g.d; ++m) {
    for (int m2 = m + 1; m2 <= g.d; ++m2) {
      TcPlan pl;
      if (!fill_plan(g, R, m, m2, want, pl)) continue;
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

struct WsLayout {
  size_t a1, a2, slots, tpart, pm, qc, ts, wl, wr, oms, total;
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
  w.wl = take(static_cast<size_t>(pl.M) * pl.R * sizeof(float));
  w.wr = take(static_cast<size_t>(pl.C) * pl.R * sizeof(float));
  w.oms = take(static_cast<size_t>(pl.S) * pl.R * sizeof(float));
  w.total = off;
  return w;
}

}  // namespace

bool tc_sketch_supported(const Dims& g, int R, const bool* want) {
  if (!device_is_sm100() || !get_encode()) return false;
  TcPlan pl;
  return choose_plan(g, R, want, pl);
}

size_t tc_sketch_ws_bytes(const Dims& g, int R, const bool* want) {
  TcPlan pl;
  if (!choose_plan(g, R, want, pl)) return 0;
  return ws_layout(pl).total;
}

int tc_sketch(const float* X, const Dims& g, const OmegaPtrs& om, int R, const bool* want, float* const* Y, Arena& ar,
              cudaStream_t s) {
  TcPlan pl;
  if (!device_is_sm100() || !choose_plan(g, R, want, pl)) {
    set_error("tcgen05 sketch: unsupported shape/device");
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
  p.NS = pl.NS;
  p.NC = pl.NC;
  p.NA = pl.NA;
  p.do_p = pl.do_p;
  p.do_q = pl.do_q;
  p.do_t = pl.do_t;
  p.maxseg = pl.maxseg;
  p.tm_acc = pl.tm_acc;
  p.tm_chunk = pl.tm_chunk;
  p.sm_x = pl.sm_x;
  p.sm_bp = pl.sm_bp;
  p.sm_bq = pl.sm_bq;
  p.sm_red = pl.sm_red;
  p.sm_bar = pl.sm_bar;
  p.m = pl.m;
  p.m2 = pl.m2;
  p.d = g.d;
  for (int k = 0; k < g.d; ++k) {
    p.n[k] = g.n[k];
    p.om[k] = om.p[k];
  }
  {  // strides inside each group
    int64_t st = 1;
    for (int k = 0; k < pl.m; ++k) p.gs[k] = st, st *= g.n[k];
    st = 1;
    for (int k = pl.m; k < pl.m2; ++k) p.gs[k] = st, st *= g.n[k];
    st = 1;
    for (int k = pl.m2; k < g.d; ++k) p.gs[k] = st, st *= g.n[k];
  }
  p.partA1 = reinterpret_cast<float*>(wsb + wl.a1);
  p.partA2 = reinterpret_cast<float*>(wsb + wl.a2);
  p.slot_pair = reinterpret_cast<int*>(wsb + wl.slots);
  p.Tpart = reinterpret_cast<float*>(wsb + wl.tpart);
  float* Pm = reinterpret_cast<float*>(wsb + wl.pm);
  float* Qc = reinterpret_cast<float*>(wsb + wl.qc);
  float* Ts = reinterpret_cast<float*>(wsb + wl.ts);
  float* WL = reinterpret_cast<float*>(wsb + wl.wl);
  float* WR = reinterpret_cast<float*>(wsb + wl.wr);
  float* OmS = reinterpret_cast<float*>(wsb + wl.oms);
  p.WL = WL;
  p.WR = WR;
  p.OmS = OmS;
  {
    const char* e = getenv("KRP_TC_DEBUG");
    p.dbg = e ? atoi(e) : 0;
  }

  CUtensorMap tmap;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(pl.M), static_cast<cuuint64_t>(pl.C),
                          static_cast<cuuint64_t>(pl.S)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(pl.M) * 4, static_cast<cuuint64_t>(pl.M * pl.C) * 4};
    cuuint32_t box[3] = {32, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(X), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
      return KRP_ECUDA;
    }
  }
  // 1. Khatri-Rao tables of the three mode groups (tiny: (M + C + S) x R)
  {
    TabParams tp{};
    tp.d = g.d;
    tp.m = pl.m;
    tp.m2 = pl.m2;
    tp.R = R;
    tp.M = pl.M;
    tp.C = pl.C;
    tp.S = pl.S;
    for (int k = 0; k < g.d; ++k) {
      tp.n[k] = p.n[k];
      tp.gs[k] = p.gs[k];
      tp.om[k] = p.om[k];
    }
    tp.WL = WL;
    tp.WR = WR;
    tp.OmS = OmS;
    const int64_t nt = (pl.M + pl.C + pl.S) * R;
    tc_tables_kernel<<<static_cast<unsigned>((nt + 255) / 256), 256, 0, s>>>(tp);
    KRP_CHECK_LAUNCH();
  }
  // 2. the fused tile kernel
  auto kern = (R <= 16)   ? krp_tc_sketch_kernel<16>
              : (R <= 32) ? krp_tc_sketch_kernel<32>
              : (R <= 48) ? krp_tc_sketch_kernel<48>
                          : krp_tc_sketch_kernel<64>;
  KRP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(pl.smem_bytes)));
  prof_begin(s);
  kern<<<pl.grid, kThreads, pl.smem_bytes, s>>>(tmap, p);
  KRP_CHECK_LAUNCH();
  prof_end(s, 4.0 * static_cast<double>(g.N), 2.0 * static_cast<double>(g.N) * R * (pl.do_p + pl.do_q));
  // 3. fixed-order sum of the per-CTA partials, then the multi-TTVs of the three groups
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
    rp.do_p = pl.do_p;
    rp.do_q = pl.do_q;
    rp.do_t = pl.do_t;
    rp.partA1 = p.partA1;
    rp.partA2 = p.partA2;
    rp.Tpart = p.Tpart;
    rp.Pm = Pm;
    rp.Qc = Qc;
    rp.Ts = Ts;
    const int64_t nasm = (pl.do_p ? pl.M * R : 0) + (pl.do_q ? pl.C * R : 0) + (pl.do_t ? pl.S * R : 0);
    tc_assemble_kernel<<<static_cast<unsigned>((nasm + 255) / 256), 256, 0, s>>>(rp);
    KRP_CHECK_LAUNCH();
  }
  {
    TtvParams tv{};
    tv.d = g.d;
    tv.m = pl.m;
    tv.m2 = pl.m2;
    tv.R = R;
    tv.M = pl.M;
    tv.C = pl.C;
    tv.S = pl.S;
    int64_t nout = 0;
    for (int k = 0; k < g.d; ++k) {
      tv.n[k] = p.n[k];
      tv.gs[k] = p.gs[k];
      tv.om[k] = p.om[k];
      tv.want[k] = want[k] ? 1 : 0;
      tv.y[k] = want[k] ? Y[k] : nullptr;
      if (want[k]) nout += g.n[k] * R;
    }
    tv.Pm = Pm;
    tv.Qc = Qc;
    tv.Ts = Ts;
    tc_ttv_kernel<<<static_cast<unsigned>((nout + 255) / 256), 256, 0, s>>>(tv);
    KRP_CHECK_LAUNCH();
  }
  ar.off = mark;
  return KRP_OK;
}

}  // namespace krp
