// krp_ttm_tc.cu — the mode-1 tensor-times-matrix product on sm_100a tensor cores (3xTF32).
//
// Y = X x_1 A, i.e. Y(j, h) = Σ_i A(j, i) X(i, h) for X of I x H (first index fastest: column h of the
// mode-1 unfolding is the contiguous run X[I h, I h + I)), A of J x I (element (j, i) at A[j sj + i si]),
// Y of J x H (Y[j + J h]).  This is the first core contraction of rHOSVD (Alg. 7 line 5,
// G = X x_1 Q_1ᵀ ... x_d Q_dᵀ) and the first STHOSVD step product (Alg. 8 line 5,
// B = X x_1 Q_1ᵀ): the two passes over the full tensor outside the sketch.
//
// As a GEMM: Yᵀ (H x J) = X_(1)ᵀ (H x I, K-major: i contiguous) · Aᵀ.  M = 128 columns h per tile, N = J
// (padded to Np = round16(J) <= 64), K = I in chunks of 32 (one TMA box {32 i, 128 h}, SWIZZLE_128B,
// out-of-range i / h zero-filled).  3xTF32 with a ROUND-TO-NEAREST split: hi = rn_tf32(x) (two integer
// ops on the bits), lo = x - hi exactly (fp32), which the tensor core reads truncated to tf32; lo has
// either sign, so the truncation of lo (<= 2^-22 |x|) and the dropped lo·lo term (<= 2^-22 |x a|) have
// either sign too.  (The sketch kernel's truncation split, hi = the raw value as the tensor core reads it,
// leaves lo with the sign of x: on a positive tensor such as c5's the dropped terms then add coherently, a
// ~1e-6 relative bias of every core entry, which is the size of c5's whole Tucker error.)
//     D[0, 2Np)   = X_hi · [A_hi | A_lo]ᵀ   (N = 2Np: columns hh | hl)
//     D[Np, 2Np) += X_lo · A_hiᵀ            (N = Np: the two small cross terms share columns)
// both with the A operand in TMEM (written by the split warps).  The tensor core's fp32 accumulation into
// TMEM rounds toward zero (measured: a positive K = 512 product came out 4.6e-6 low, ~0.6 ulp per
// accumulating MMA), so the accumulators hold ONE K chunk (4 accumulating MMAs on the hh columns) and are
// drained every chunk: the epilogue warps add hh + (hl + lh) of each chunk into fp32 registers with
// round-to-nearest adds, in chunk order (the cross-term columns are 2^-11 smaller: their own rounding
// bias is negligible).  The B operand [A_hi | A_lo] of every K chunk is
// prepared once per call (a tiny kernel) as the exact shared-memory image (rows of 128 B, 128B swizzle)
// and streamed next to each X box by a bulk copy (it stays in L2: <= 1 MB).
//
// Persistent kernel, one CTA per SM, tiles of 128 columns split contiguously over the CTAs.  Warps:
// 0 TMA producer (X boxes: a deep ring released as soon as the split warps hold a box in registers),
// 10 bulk-copy producer (B images: resident when I <= 128, else a ring released by the MMAs), 1 MMA issuer
// (owns TMEM), 2-5 split (X_hi, X_lo of each chunk into TMEM, one row per thread),
// 6-9 epilogue (per-chunk accumulators -> register sums -> per-warp shared staging -> coalesced stores of
// the contiguous run Y[J h0, J (h0 + 32))).  Chunk accumulators are double-buffered in TMEM so a chunk's
// drain overlaps the next chunk's MMAs.  Every element of X is read from HBM once; the sum over i runs in a fixed order, so
// the result is deterministic.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "krp_common.cuh"
#include "krp_internal.h"
#include "sm100.cuh"

namespace krp {
namespace {
using namespace sm100;

constexpr int kT0Threads = 11 * 32;
constexpr int kT0Rows = 128;   // tile: 128 columns h
constexpr int kT0K = 32;       // K chunk: one 128-byte row of the TMA box
constexpr int kT0SlotCols = 64;  // TMEM columns of one chunk slot: X_hi [0, 32), X_lo [32, 64)
constexpr int kT0MaxNC = 4;    // chunk slots (X_hi | X_lo), as many as TMEM leaves room for
constexpr int kT0NA = 2;       // chunk accumulator stages, 2 Np columns each (hh | hl + lh)
constexpr int kT0MaxJ = 64;

struct Ttm0Params {
  int64_t H;
  int I, J, Np, nk;  // nk = ceil(I / 32) K chunks per tile
  int64_t T;         // tiles = ceil(H / 128)
  int NSX, NSB;      // smem stages: X boxes (16 KB), B images (resident when nk <= NSB)
  int NC;            // TMEM chunk slots
  uint32_t sm_x, sm_b, sm_stg, sm_bar;
  uint32_t b_bytes;  // one B image chunk: 2 Np rows x 128 B
  const float* Bimg; // [nk][2 Np][32] swizzled: rows [0, Np) A_hi, [Np, 2Np) A_lo
  float* Y;
  int64_t H1;        // > 0: permuted output Y[h1 + H1 (j + J h2)] for h = h1 + H1 h2 (else Y[j + J h])
};

// round to the nearest tf32 (ties away from zero); the result has its 13 low mantissa bits clear
__device__ __forceinline__ uint32_t tf32_rn_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// round to the nearest tf32 on the bits (ties away from zero: +half an ulp of tf32 on the magnitude, then
// clear the 13 low mantissa bits); finite inputs (an infinity becomes a NaN, which it would produce anyway)
__device__ __forceinline__ uint32_t tf32_rn_fast(uint32_t u) { return (u + 0x1000u) & 0xFFFFE000u; }

// B image: element (row n, k) of chunk kc at byte kc * 2Np*128 + sw128_offset(n, k)
__global__ void ttm0_bimg_kernel(const float* __restrict__ A, int J, int I, int64_t sj, int64_t si, int Np, int nk,
                                 float* __restrict__ img) {
  const int64_t total = static_cast<int64_t>(nk) * 2 * Np * kT0K;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e % kT0K);
    const int64_t rn = e / kT0K;
    const int n = static_cast<int>(rn % (2 * Np));
    const int kc = static_cast<int>(rn / (2 * Np));
    const int j = n < Np ? n : n - Np;
    const int i = kc * kT0K + k;
    const float v = (j < J && i < I) ? A[j * sj + i * si] : 0.f;
    const float hi = __uint_as_float(tf32_rn_bits(v));
    const float out = n < Np ? hi : __uint_as_float(tf32_rn_bits(v - hi));
    const size_t byte = static_cast<size_t>(kc) * 2 * Np * 128 + sw128_offset(static_cast<uint32_t>(n), static_cast<uint32_t>(k));
    img[byte / 4] = out;
  }
}

__device__ __forceinline__ void t0_sts(uint32_t saddr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(saddr), "f"(v) : "memory");
}
__device__ __forceinline__ float t0_lds(uint32_t saddr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr) : "memory");
  return v;
}

#define T0WAIT(bar, par) mbar_wait_hint((bar), (par), 10000000u)

__global__ void __launch_bounds__(kT0Threads, 1)
    ttm0_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Ttm0Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xs = smem + p.sm_x;
  uint8_t* bs = smem + p.sm_b;
  float* stg = reinterpret_cast<float*>(smem + p.sm_stg);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.sm_bar);
  uint64_t* full_x = bars;
  uint64_t* empty_x = full_x + p.NSX;
  uint64_t* full_b = empty_x + p.NSX;
  uint64_t* empty_b = full_b + p.NSB;
  uint64_t* lo_full = empty_b + p.NSB;
  uint64_t* lo_free = lo_full + kT0MaxNC;
  uint64_t* acc_full = lo_free + kT0MaxNC;
  uint64_t* acc_empty = acc_full + kT0NA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kT0NA);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.NSX; ++i) {
      mbar_init(&full_x[i], 1);
      mbar_init(&empty_x[i], 4);  // the split warps' reads (the MMAs read X from TMEM)
    }
    for (int i = 0; i < p.NSB; ++i) {
      mbar_init(&full_b[i], 1);
      mbar_init(&empty_b[i], 1);  // the MMAs' commit
    }
    for (int i = 0; i < p.NC; ++i) {
      mbar_init(&lo_full[i], 4);
      mbar_init(&lo_free[i], 1);
    }
    for (int i = 0; i < kT0NA; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tm_slot = static_cast<uint32_t>(kT0NA * 2 * p.Np);  // chunk slots after the accumulators

  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * p.T / gridDim.x;
  const int64_t t1 = static_cast<int64_t>(blockIdx.x + 1) * p.T / gridDim.x;
  const int nk = p.nk;

  const bool b_resident = nk <= p.NSB;  // every B chunk loaded once, never released
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: X boxes
    if (elect_one()) {
      tma_prefetch_desc(&tmap);
      const uint64_t pol = policy_evict_first();
      int st = 0;
      uint32_t ph = 0;
      for (int64_t t = t0; t < t1; ++t) {
        for (int kc = 0; kc < nk; ++kc) {
          T0WAIT(&empty_x[st], ph ^ 1);
          mbar_arrive_expect_tx(&full_x[st], kT0Rows * 128);
          tma_load_2d(xs + st * (kT0Rows * 128), &tmap, &full_x[st], kc * kT0K, static_cast<int32_t>(t * kT0Rows), pol);
          if (++st == p.NSX) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ bulk-copy producer: B images
    if (elect_one()) {
      const uint8_t* img = reinterpret_cast<const uint8_t*>(p.Bimg);
      if (b_resident) {
        for (int kc = 0; kc < nk; ++kc) {
          mbar_arrive_expect_tx(&full_b[kc], p.b_bytes);
          bulk_copy_g2s(bs + kc * p.b_bytes, img + static_cast<size_t>(kc) * p.b_bytes, p.b_bytes, &full_b[kc]);
        }
      } else {
        int st = 0;
        uint32_t ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
          for (int kc = 0; kc < nk; ++kc) {
            T0WAIT(&empty_b[st], ph ^ 1);
            mbar_arrive_expect_tx(&full_b[st], p.b_bytes);
            bulk_copy_g2s(bs + st * p.b_bytes, img + static_cast<size_t>(kc) * p.b_bytes, p.b_bytes, &full_b[st]);
            if (++st == p.NSB) {
              st = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const bool leader = elect_one();
    const uint32_t idesc_cat = make_idesc_tf32(128, 2 * p.Np, 0, 0);
    const uint32_t idesc_lo = make_idesc_tf32(128, p.Np, 0, 0);
    const uint64_t bdesc0 = make_smem_desc(smem_u32(bs), 0, 1024, kLayoutSW128);
    int st = 0, cs = 0, as = 0;
    uint32_t ph = 0, cph = 0, aph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      for (int kc = 0; kc < nk; ++kc) {
        if (b_resident) st = kc;
        T0WAIT(&acc_empty[as], aph ^ 1);
        T0WAIT(&full_b[st], b_resident ? 0u : ph);
        T0WAIT(&lo_full[cs], cph);
        tc_fence_after();
        const uint32_t d1 = tbase + static_cast<uint32_t>(as * 2 * p.Np), d2 = d1 + p.Np;
        const uint64_t bd = bdesc0 + ((static_cast<uint64_t>(st) * p.b_bytes) >> 4);
        const uint32_t thi = tbase + tm_slot + static_cast<uint32_t>(cs * kT0SlotCols);
        if (leader) {
#pragma unroll
          for (int ks = 0; ks < kT0K / 8; ++ks) {  // K = 8 per MMA: +32 B on the B descriptor's start address
            mma_tf32_ts(d1, thi + 8 * ks, bd + ks * 2, idesc_cat, ks ? 1u : 0u);       // hi x [A_hi | A_lo]
            mma_tf32_ts(d2, thi + 32 + 8 * ks, bd + ks * 2, idesc_lo, 1u);             // lo x A_hi
          }
          if (!b_resident) mma_commit(&empty_b[st]);
          mma_commit(&lo_free[cs]);
          mma_commit(&acc_full[as]);
        }
        __syncwarp();
        if (!b_resident && ++st == p.NSB) {
          st = 0;
          ph ^= 1;
        }
        if (++cs == p.NC) {
          cs = 0;
          cph ^= 1;
        }
        if (++as == kT0NA) {
          as = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ split: X_hi, X_lo -> TMEM (row = lane)
    const uint32_t q = warp & 3u;
    const uint32_t row = 32u * q + lane;
    const uint32_t lane_off = (32u * q) << 16;
    const uint32_t rx = row & 7u;
    int st = 0, cs = 0;
    uint32_t ph = 0, cph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      for (int kc = 0; kc < nk; ++kc) {
        T0WAIT(&full_x[st], ph);
        T0WAIT(&lo_free[cs], cph ^ 1);
        tc_fence_after();
        const uint32_t rowa = smem_u32(xs) + static_cast<uint32_t>(st) * (kT0Rows * 128) + row * 128u;
        uint32_t v[kT0K];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float a0, a1, a2, a3;
          lds_v4(rowa + ((static_cast<uint32_t>(c) ^ rx) << 4), a0, a1, a2, a3);
          v[4 * c] = __float_as_uint(a0), v[4 * c + 1] = __float_as_uint(a1);
          v[4 * c + 2] = __float_as_uint(a2), v[4 * c + 3] = __float_as_uint(a3);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_x[st]);  // the box is in registers: release it to the producer
        uint32_t hv[kT0K];
#pragma unroll
        for (int k = 0; k < kT0K; k += 2) {
          hv[k] = tf32_rn_fast(v[k]);
          hv[k + 1] = tf32_rn_fast(v[k + 1]);
          const float2 l = f2_sub(make_float2(__uint_as_float(v[k]), __uint_as_float(v[k + 1])),
                                  make_float2(__uint_as_float(hv[k]), __uint_as_float(hv[k + 1])));
          v[k] = __float_as_uint(l.x);
          v[k + 1] = __float_as_uint(l.y);
        }
        const uint32_t slot = tbase + lane_off + tm_slot + static_cast<uint32_t>(cs * kT0SlotCols);
        tmem_st<32>(slot, hv);
        tmem_st<32>(slot + 32, v);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&lo_full[cs]);
        if (++st == p.NSX) {
          st = 0;
          ph ^= 1;
        }
        if (++cs == p.NC) {
          cs = 0;
          cph ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3u;
    const uint32_t lane_off = (32u * q) << 16;
    const int J = p.J, Np = p.Np;
    const uint32_t wsa = smem_u32(stg + q * 32 * kT0MaxJ);  // this warp's 32 rows: the contiguous run Y[J h0, ...)
    int as = 0;
    uint32_t aph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      float acc[kT0MaxJ];
#pragma unroll
      for (int j = 0; j < kT0MaxJ; ++j) acc[j] = 0.f;
      for (int kc = 0; kc < nk; ++kc) {
        T0WAIT(&acc_full[as], aph);
        tc_fence_after();
        const uint32_t d1 = tbase + lane_off + static_cast<uint32_t>(as * 2 * Np);
#pragma unroll
        for (int c = 0; c < kT0MaxJ; c += 16) {
          if (c < Np) {
            uint32_t hh[16], hl[16];
            tmem_ld<16>(d1 + c, hh);
            tmem_ld<16>(d1 + Np + c, hl);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; k += 2) {
              const float2 t = f2_add(make_float2(__uint_as_float(hh[k]), __uint_as_float(hh[k + 1])),
                                      make_float2(__uint_as_float(hl[k]), __uint_as_float(hl[k + 1])));
              const float2 a2 = f2_add(make_float2(acc[c + k], acc[c + k + 1]), t);
              acc[c + k] = a2.x;
              acc[c + k + 1] = a2.y;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[as]);
        if (++as == kT0NA) {
          as = 0;
          aph ^= 1;
        }
      }
      const int64_t h0 = t * kT0Rows + 32 * q;
      if (p.H1 > 0) {
        // permuted output Y[h1 + H1 (j + J h2)], h = h1 + H1 h2: for each j the warp's 32 consecutive rows are
        // (up to an h2 wrap) 32 consecutive floats, stored straight from the registers
        const int64_t h = h0 + lane;
        if (h < p.H) {
          const int64_t h2 = h / p.H1, h1 = h - h2 * p.H1;
          float* out = p.Y + h1 + p.H1 * static_cast<int64_t>(J) * h2;
#pragma unroll
          for (int j = 0; j < kT0MaxJ; ++j)
            if (j < J) out[p.H1 * j] = acc[j];
        }
      } else {
        __syncwarp();  // the previous tile's copy-out of the staging rows is done
        const uint32_t wrow = wsa + lane * static_cast<uint32_t>(J) * 4u;
#pragma unroll
        for (int j = 0; j < kT0MaxJ; ++j)
          if (j < J) t0_sts(wrow + 4u * j, acc[j]);
        __syncwarp();
        const int64_t nr = min(static_cast<int64_t>(32), p.H - h0);
        if (nr > 0) {
          float* out = p.Y + static_cast<int64_t>(J) * h0;
          const int n = static_cast<int>(nr) * J;
          for (int e = static_cast<int>(lane); e < n; e += 32) out[e] = t0_lds(wsa + 4u * e);
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

int round16i(int v) { return (v + 15) / 16 * 16; }

}  // namespace

bool ttm0_tc_ok(const float* X, int64_t I, int64_t H, int J) {
  return tc_device_ok() && J >= 1 && J <= kT0MaxJ && I >= 1 && I % 4 == 0 && I < (int64_t(1) << 31) && H >= 1 &&
         H < (int64_t(1) << 31) && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
}

size_t ttm0_tc_ws_bytes(int64_t I, int J) {
  const int64_t nk = (I + kT0K - 1) / kT0K;
  return align_up(static_cast<size_t>(nk) * 2 * round16i(J) * kT0K * sizeof(float), 256);
}

int ttm0_tc(const float* X, int64_t I, int64_t H, const float* A, int J, int64_t sj, int64_t si, float* Y, Arena& ar,
            cudaStream_t s, int64_t H1) {
  if (!ttm0_tc_ok(X, I, H, J)) {
    set_error("ttm0_tc: unsupported shape or device (I=%lld H=%lld J=%d)", static_cast<long long>(I),
              static_cast<long long>(H), J);
    return KRP_EUNSUPPORTED;
  }
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encode_fn());
  Ttm0Params p{};
  p.H = H;
  p.I = static_cast<int>(I);
  p.J = J;
  p.Np = round16i(J);
  p.nk = static_cast<int>((I + kT0K - 1) / kT0K);
  p.T = (H + kT0Rows - 1) / kT0Rows;
  p.b_bytes = static_cast<uint32_t>(2 * p.Np * 128);
  const size_t mark = ar.off;
  float* img = ar.take<float>(static_cast<size_t>(p.nk) * 2 * p.Np * kT0K);
  if (ar.overflow()) {
    set_error("workspace too small for the mode-1 TTM");
    return KRP_ENOMEM;
  }
  p.Bimg = img;
  p.Y = Y;
  p.H1 = (H1 > 0 && H % H1 == 0) ? H1 : 0;
  // shared memory (~208 KB): X boxes (16 KB each), B images (all of them when nk <= 4, else a ring of 3),
  // the epilogue staging, barriers
  const uint32_t stg_bytes = 4 * 32 * kT0MaxJ * 4;
  p.NSB = p.nk <= 4 ? p.nk : 3;
  const uint32_t budget = 208 * 1024 - stg_bytes - 1024 - p.NSB * p.b_bytes;
  p.NSX = static_cast<int>(std::min<uint32_t>(10, budget / (kT0Rows * 128)));
  p.sm_x = 0;
  p.sm_b = p.NSX * kT0Rows * 128;
  p.sm_stg = p.sm_b + p.NSB * p.b_bytes;
  p.sm_bar = p.sm_stg + stg_bytes;
  const uint32_t smem_bytes = p.sm_bar + (2 * p.NSX + 2 * p.NSB + 2 * kT0MaxNC + 2 * kT0NA) * 8 + 16 + 1024;
  p.NC = std::min(kT0MaxNC, (512 - kT0NA * 2 * p.Np) / kT0SlotCols);  // TMEM: 2 x 2 Np + NC x 64 <= 512

  CUtensorMap tmap;
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(I), static_cast<cuuint64_t>(H)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(I) * 4};
    cuuint32_t box[2] = {kT0K, kT0Rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
      return KRP_ECUDA;
    }
  }
  {
    const int64_t total = static_cast<int64_t>(p.nk) * 2 * p.Np * kT0K;
    const unsigned nb = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 1024));
    ttm0_bimg_kernel<<<nb, 256, 0, s>>>(A, J, p.I, sj, si, p.Np, p.nk, img);
    KRP_CHECK_LAUNCH();
  }
  KRP_CHECK_CUDA(cudaFuncSetAttribute(ttm0_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem_bytes)));
  const int grid = static_cast<int>(std::min<int64_t>(p.T, device_sms()));
  ttm0_tc_kernel<<<grid, kT0Threads, smem_bytes, s>>>(tmap, p);
  KRP_CHECK_LAUNCH();
  ar.off = mark;
  return KRP_OK;
}

}  // namespace krp
