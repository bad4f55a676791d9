// tcprobe.cu — sm_100a probes that fix the design parameters of the fused KRP
// sketch kernel (DESIGN.md §"Measured facts"):
//   (1) semantics: does tcgen05.mma kind::tf32 read a raw fp32 operand by
//       truncation or by round-to-nearest?  Are our UMMA descriptors for the
//       TMA SWIZZLE_128B tile right in BOTH views (MN-major A for P = X·W_R and
//       K-major A for Q = Xᵀ·W_L)?  Same for A staged in TMEM (tcgen05.st).
//   (2) throughput: cycles per tcgen05.mma (M=128, K=8) for N in {16..128},
//       SS (A K-major / MN-major) and TS (A in TMEM), alone and with 4 warps
//       streaming shared memory at the same time (is the UMMA operand read
//       path shared with LDS bandwidth?).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tcprobe tcprobe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"

using namespace sm100;

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e = (x);                                                                       \
    if (e != cudaSuccess) {                                                                    \
      fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

// ------------------------------------------------------------------ (1) semantics
constexpr int kN = 48;  // sketch width used in the semantics probe
struct alignas(1024) SemSmem {
  float xtile[4][128][32];  // 4 TMA boxes {32 i1 x 128 c}, SWIZZLE_128B
  float b1[4][kN][32];      // W_R: K = c (128) x N, K-major SW128
  float b2[4][kN][32];      // W_L: K = i1 (128) x N
  uint64_t bar_tma, bar_mma;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128, 1)
    sem_kernel(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ W1,  // [128 c][N]
               const float* __restrict__ W2,                                           // [128 i1][N]
               const float* __restrict__ Xg,  // [c][i1] i1 fastest (same as tensor memory order)
               float* __restrict__ out,       // 4 x [128][N]
               int mn_variant)
{
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SemSmem& s = *reinterpret_cast<SemSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc<512>(&s.tmem_base);
  if (tid == 0) {
    mbar_init(&s.bar_tma, 1);
    mbar_init(&s.bar_mma, 1);
    fence_barrier_init();
  }
  // B operands, K-major SW128: element (n, k) at [k/32][n] row, swizzled chunk.
  for (int idx = tid; idx < 128 * kN; idx += 128) {
    int k = idx / kN, n = idx % kN;
    uint8_t* base1 = reinterpret_cast<uint8_t*>(&s.b1[k >> 5][0][0]);
    uint8_t* base2 = reinterpret_cast<uint8_t*>(&s.b2[k >> 5][0][0]);
    *reinterpret_cast<float*>(base1 + sw128_offset(n, k & 31)) = W1[k * kN + n];
    *reinterpret_cast<float*>(base2 + sw128_offset(n, k & 31)) = W2[k * kN + n];
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s.tmem_base;
  if (tid == 0) {
    mbar_arrive_expect_tx(&s.bar_tma, 4 * 128 * 32 * 4);
    for (int j = 0; j < 4; ++j) tma_load_2d(&s.xtile[j][0][0], &tmap, &s.bar_tma, 32 * j, 0, policy_evict_first());
  }
  mbar_wait(&s.bar_tma, 0);
  tc_fence_after();
  const uint32_t idesc_p = make_idesc_tf32(128, kN, /*a MN*/ 1, 0);
  const uint32_t idesc_q = make_idesc_tf32(128, kN, 0, 0);
  const uint32_t xb = smem_u32(&s.xtile[0][0][0]);
  const uint32_t b1b = smem_u32(&s.b1[0][0][0]), b2b = smem_u32(&s.b2[0][0][0]);
  if (tid == 0) {
    for (int kk = 0; kk < 16; ++kk) {
      // P: A = X(i1, c), M = i1 (MN-major, LBO = box stride 16 KB, SBO = 8 c-rows = 1 KB), K = c.
      uint64_t a = mn_variant == 0 ? make_smem_desc(xb + kk * 1024, 16384, 1024, kLayoutSW128)
                                   : make_smem_desc(xb + kk * 1024, 1024, 16384, kLayoutSW128);
      uint64_t b = make_smem_desc(b1b + (kk >> 2) * (kN * 128) + (kk & 3) * 32, 0, 1024, kLayoutSW128);
      mma_tf32_ss(tbase + 0, a, b, idesc_p, kk > 0);
    }
    for (int kk = 0; kk < 16; ++kk) {
      // Q: A = X(i1, c)^T, M = c (rows of 128 B), K = i1 (K-major, 32 B steps inside the atom).
      uint64_t a = make_smem_desc(xb + (kk >> 2) * 16384 + (kk & 3) * 32, 0, 1024, kLayoutSW128);
      uint64_t b = make_smem_desc(b2b + (kk >> 2) * (kN * 128) + (kk & 3) * 32, 0, 1024, kLayoutSW128);
      mma_tf32_ss(tbase + 64, a, b, idesc_q, kk > 0);
    }
    mma_commit(&s.bar_mma);
  }
  mbar_wait(&s.bar_mma, 0);
  tc_fence_after();
  // TS path: stage A in TMEM.  P-layout: lane i1, column c (cols 128..255);
  //                             Q-layout: lane c, column i1 (cols 256..383).
  {
    const uint32_t row = tid;  // lane
    for (int c0 = 0; c0 < 128; c0 += 16) {
      uint32_t rp[16], rq[16];
      for (int j = 0; j < 16; ++j) {
        rp[j] = __float_as_uint(Xg[(c0 + j) * 128 + row]);  // X(i1=row, c=c0+j)
        rq[j] = __float_as_uint(Xg[row * 128 + c0 + j]);    // X(i1=c0+j, c=row)
      }
      tmem_st16(tbase + ((warp * 32) << 16) + 128 + c0, rp);
      tmem_st16(tbase + ((warp * 32) << 16) + 256 + c0, rq);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = make_idesc_tf32(128, kN, 0, 0);
    for (int kk = 0; kk < 16; ++kk) {
      uint64_t b = make_smem_desc(b1b + (kk >> 2) * (kN * 128) + (kk & 3) * 32, 0, 1024, kLayoutSW128);
      mma_tf32_ts(tbase + 384, tbase + 128 + kk * 8, b, idesc, kk > 0);
    }
    for (int kk = 0; kk < 16; ++kk) {
      uint64_t b = make_smem_desc(b2b + (kk >> 2) * (kN * 128) + (kk & 3) * 32, 0, 1024, kLayoutSW128);
      mma_tf32_ts(tbase + 448, tbase + 256 + kk * 8, b, idesc, kk > 0);
    }
    mma_commit(&s.bar_mma);
  }
  mbar_wait(&s.bar_mma, 1);
  tc_fence_after();
  const int cols[4] = {0, 64, 384, 448};
  for (int o = 0; o < 4; ++o) {
    for (int n0 = 0; n0 < kN; n0 += 8) {
      float v[8];
      tmem_ld8(tbase + ((warp * 32) << 16) + cols[o] + n0, v);
      tmem_ld_wait();
      for (int j = 0; j < 8; ++j) out[o * 128 * kN + tid * kN + n0 + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ (2) throughput
struct alignas(1024) TpSmem {
  float a[4][128][32];   // 64 KB A tile (SW128)
  float b[4][128][32];   // up to N=128 B (K-major SW128)
  float4 junk[2048];     // 32 KB region hammered by the LDS warps
  uint64_t bar[2];
  uint32_t tmem_base;
};

template <int MODE, int N, int HAMMER>
__global__ void __launch_bounds__(256, 1) tp_kernel(int iters, unsigned long long* cycles, float* sink) {
  // MODE 0: SS, A K-major; 1: SS, A MN-major; 2: TS (A in TMEM)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TpSmem& s = *reinterpret_cast<TpSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc<512>(&s.tmem_base);
  if (tid == 0) {
    mbar_init(&s.bar[0], 1);
    mbar_init(&s.bar[1], 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 4 * 128 * 32; i += 256) {
    (&s.a[0][0][0])[i] = 1.0f;
    (&s.b[0][0][0])[i] = 1.0f;
  }
  for (int i = tid; i < 2048; i += 256) s.junk[i] = make_float4(i, 1, 2, 3);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s.tmem_base;
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t ab = smem_u32(&s.a[0][0][0]), bb = smem_u32(&s.b[0][0][0]);
      const uint32_t idesc = make_idesc_tf32(128, N, MODE == 1 ? 1 : 0, 0);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        const int slot = it & 1;
        if (it >= 2) mbar_wait(&s.bar[slot], ((it >> 1) - 1) & 1);
        tc_fence_after();
        for (int kk = 0; kk < 16; ++kk) {
          uint64_t b = make_smem_desc(bb + (kk >> 2) * (N * 128) + (kk & 3) * 32, 0, 1024, kLayoutSW128);
          const uint32_t d = tbase + slot * 128;
          if (MODE == 0) {
            uint64_t a = make_smem_desc(ab + (kk >> 2) * 16384 + (kk & 3) * 32, 0, 1024, kLayoutSW128);
            mma_tf32_ss(d, a, b, idesc, kk > 0);
          } else if (MODE == 1) {
            uint64_t a = make_smem_desc(ab + kk * 1024, 16384, 1024, kLayoutSW128);
            mma_tf32_ss(d, a, b, idesc, kk > 0);
          } else if (MODE == 2) {
            mma_tf32_ts(d, tbase + 256 + (kk & 15) * 8, b, idesc, kk > 0);
          } else if (MODE == 3) {
            const uint32_t id80 = make_idesc_tf32(128, 80, 0, 0);
            mma_tf32_ts(d, tbase + 256 + (kk & 15) * 8, b, (kk & 1) ? idesc : id80, kk > 0);
          } else if (MODE == 6 || MODE == 7 || MODE == 8) {
            // kernel-like: per K-step 3 MMAs (hi.hi, hi.lo with B at +5120 B, lo.hi), two GEMMs (D at 0 / 48)
            // MODE 6: A at 256.., D at slot*128 (+0/+48) ; MODE 7: kernel TMEM layout (A at 192.., D at slot*96)
            // MODE 8: MODE 7 but only one GEMM (D at slot*96)
            const uint32_t abase = (MODE == 6) ? 256u : 192u;
            const uint32_t dslot = (MODE == 6) ? slot * 128 : slot * 96;
            const uint32_t acol = abase + (kk & 1) * 64 + ((kk >> 1) & 1) * 8;
            uint64_t bl = make_smem_desc(bb + (kk >> 2) * (N * 128) + (kk & 3) * 32 + 5120, 0, 1024, kLayoutSW128);
            for (int g = 0; g < (MODE == 8 ? 1 : 2); ++g) {
              const uint32_t dd = tbase + dslot + g * 48;
              mma_tf32_ts(dd, tbase + acol + g * 32, b, idesc, kk > 0);
              mma_tf32_ts(dd, tbase + acol + g * 32, bl, idesc, 1);
              mma_tf32_ts(dd, tbase + acol + g * 32 + 16, b, idesc, 1);
            }
          } else if (MODE == 4) {
            uint64_t a = make_smem_desc(ab + (kk >> 2) * 16384 + (kk & 3) * 32, 0, 1024, kLayoutSW128);
            const uint32_t idf = (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                         :: "r"(d), "l"(a), "l"(b), "r"(idf), "r"((uint32_t)(kk > 0)) : "memory");
          } else {
            const uint32_t idf = (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                         :: "r"(d), "r"(tbase + 256 + (kk & 15) * 8), "l"(b), "r"(idf), "r"((uint32_t)(kk > 0)) : "memory");
          }
        }
        mma_commit(&s.bar[slot]);
      }
      mbar_wait(&s.bar[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
      if (iters >= 2) mbar_wait(&s.bar[(iters - 2) & 1], ((iters - 2) >> 1) & 1);
      long long t1 = clock64();
      cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    __syncwarp();
  } else if (HAMMER && warp >= 4) {
    // 4 warps stream LDS.128 over 32 KB for roughly the same duration.
    float4 acc = make_float4(0, 0, 0, 0);
    const int reps = iters * 16 * N / 64;
    long long h0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 8
      for (int i = 0; i < 16; ++i) {
        float4 v = s.junk[((tid & 127) + i * 128 + r) & 2047];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    sink[blockIdx.x * 256 + tid] = acc.x + acc.y + acc.z + acc.w;
    if ((tid & 127) == 0) cycles[gridDim.x + blockIdx.x] = (unsigned long long)(clock64() - h0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

__global__ void __launch_bounds__(128, 1) tmem_bw_kernel(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t tbase_s;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s + ((warp * 32) << 16);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[16];
#pragma unroll
    for (int c = 0; c < 256; c += 16) {
      tmem_ld16(tb + c, v);
      tmem_ld_wait();
      acc += v[0] + v[15];
    }
  }
  long long t1 = clock64();
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(acc + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 256; c += 16) tmem_st16(tb + 256 + c, r);
    tmem_st_wait();
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    cycles[2 * blockIdx.x] = t1 - t0;
    cycles[2 * blockIdx.x + 1] = t2 - t1;
  }
  sink[blockIdx.x * 128 + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase_s);
}

void run_tmem_bw(int nsm) {
  unsigned long long* dcyc;
  float* sink;
  CK(cudaMalloc(&dcyc, 2 * nsm * sizeof(unsigned long long)));
  CK(cudaMalloc(&sink, nsm * 128 * sizeof(float)));
  const int iters = 1000;
  tmem_bw_kernel<<<nsm, 128>>>(10, dcyc, sink);
  tmem_bw_kernel<<<nsm, 128>>>(iters, dcyc, sink);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> c(2 * nsm);
  CK(cudaMemcpy(c.data(), dcyc, 2 * nsm * 8, cudaMemcpyDeviceToHost));
  const double bytes = (double)iters * 256 * 128 * 4;  // per CTA
  printf("TMEM ld (4 warps, x16 + wait each): %.1f B/cyc/SM ; TMEM st x16: %.1f B/cyc/SM\n", bytes / c[0], bytes / c[1]);
}

// Chunked issue like the sketch kernel: per chunk 12 MMAs (2 K-steps x 2 GEMMs x 3), then commit to
// chunk_empty[c]; before a chunk, wait (on chunk_empty of the chunk NC earlier) + fence.
template <int NC, int WAITMODE>
__global__ void __launch_bounds__(256, 1) chunk_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TpSmem& s = *reinterpret_cast<TpSmem*>(smem_raw);
  __shared__ uint64_t cb[8];
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc<512>(&s.tmem_base);
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&cb[i], 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 4 * 128 * 32; i += 256) (&s.b[0][0][0])[i] = 1.0f;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s.tmem_base;
  if (warp == 0 && elect_one()) {
    const uint32_t bb = smem_u32(&s.b[0][0][0]);
    const uint32_t idesc = make_idesc_tf32(128, 48, 0, 0);
    long long t0 = clock64();
    int nchunks = iters * 8;
    for (int c = 0; c < nchunks; ++c) {
      const int st = c % NC;
      if (WAITMODE == 1 && c >= NC) mbar_wait(&cb[st], ((c / NC) - 1) & 1);
      tc_fence_after();
      for (int ks = 0; ks < 2; ++ks) {
        const int kk = (c * 2 + ks) & 15;
        uint64_t b = make_smem_desc(bb + (kk >> 2) * (48 * 128) + (kk & 3) * 32, 0, 1024, kLayoutSW128);
        uint64_t bl = make_smem_desc(bb + (kk >> 2) * (48 * 128) + (kk & 3) * 32 + 5120, 0, 1024, kLayoutSW128);
        const uint32_t acol = 192 + st * 64 + ks * 8;
        for (int g = 0; g < 2; ++g) {
          const uint32_t dd = tbase + ((c / 8) & 1) * 96 + g * 48;
          mma_tf32_ts(dd, tbase + acol + g * 32, b, idesc, kk > 0);
          mma_tf32_ts(dd, tbase + acol + g * 32, bl, idesc, 1);
          mma_tf32_ts(dd, tbase + acol + g * 32 + 16, b, idesc, 1);
        }
      }
      mma_commit(&cb[st]);
    }
    for (int c = nchunks - NC; c < nchunks; ++c) mbar_wait(&cb[c % NC], (c / NC) & 1);
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int NC, int WAITMODE>
void run_chunk(const char* name, int nsm) {
  auto k = chunk_kernel<NC, WAITMODE>;
  size_t smem = sizeof(TpSmem) + 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned long long* dcyc;
  CK(cudaMalloc(&dcyc, nsm * sizeof(unsigned long long)));
  k<<<nsm, 256, smem>>>(10, dcyc);
  CK(cudaDeviceSynchronize());
  k<<<nsm, 256, smem>>>(500, dcyc);
  CK(cudaDeviceSynchronize());
  unsigned long long c;
  CK(cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost));
  printf("%-40s NC=%d: %.1f cyc/chunk (12 MMAs), %.1f cyc/mma\n", name, NC, c / 4000.0, c / 48000.0);
  cudaFree(dcyc);
}

template <int MODE, int N, int HAMMER>
void run_tp(const char* name, int nsm) {
  auto k = tp_kernel<MODE, N, HAMMER>;
  size_t smem = sizeof(TpSmem) + 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned long long* dcyc;
  float* sink;
  CK(cudaMalloc(&dcyc, 2 * nsm * sizeof(unsigned long long)));
  CK(cudaMemset(dcyc, 0, 2 * nsm * sizeof(unsigned long long)));
  CK(cudaMalloc(&sink, nsm * 256 * sizeof(float)));
  const int iters = 2000;
  k<<<nsm, 256, smem>>>(10, dcyc, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<nsm, 256, smem>>>(iters, dcyc, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> cyc(2 * nsm);
  CK(cudaMemcpy(cyc.data(), dcyc, 2 * nsm * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  double mx = 0, hx = 0;
  for (int i = 0; i < nsm; ++i) mx = fmax(mx, (double)cyc[i]);
  for (int i = 0; i < nsm; ++i) hx = fmax(hx, (double)cyc[nsm + i]);
  if (HAMMER) {
    const double bytes = (double)(iters * 16 * N / 64) * 16 * 16 * 128;
    printf("   hammer: %.1f B/cyc/SM LDS over %.0f cyc (mma region %.0f cyc)\n", bytes / hx, hx, mx);
  }
  const double n_mma = (double)iters * 16 * ((MODE == 6 || MODE == 7) ? 6 : (MODE == 8 ? 3 : 1));
  const double flops = 2.0 * 128 * N * ((MODE >= 4) ? 16 : 8) * n_mma * nsm;
  printf("%-28s N=%3d hammer=%d  cyc/mma=%7.2f  (floor %5.1f)  TF32 TFLOP/s=%7.1f  clk=%.0f MHz\n", name, N,
         HAMMER, mx / n_mma, 128.0 * N / 256.0, flops / (ms * 1e-3) / 1e12, mx / (ms * 1e-3) / 1e6);
  cudaFree(dcyc);
  cudaFree(sink);
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static float tf32_trunc(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static float tf32_rn(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;  // round half up on magnitude (ties away)
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s, %d SMs, smem/block optin %zu, L2 %d\n", prop.name, prop.multiProcessorCount,
         prop.sharedMemPerBlockOptin, prop.l2CacheSize);
  // ---------------- semantics
  srand(1234);
  std::vector<float> X(128 * 128), W1(128 * kN), W2(128 * kN);
  auto rnd = []() { return (float)((rand() / (double)RAND_MAX) * 2.0 - 1.0) * 1.2345678f; };
  for (auto& v : X) v = rnd();
  for (auto& v : W1) v = rnd();
  for (auto& v : W2) v = rnd();
  float *dX, *dW1, *dW2, *dout;
  CK(cudaMalloc(&dX, X.size() * 4));
  CK(cudaMalloc(&dW1, W1.size() * 4));
  CK(cudaMalloc(&dW2, W2.size() * 4));
  CK(cudaMalloc(&dout, 4 * 128 * kN * 4));
  CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dW1, W1.data(), W1.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dW2, W2.data(), W2.size() * 4, cudaMemcpyHostToDevice));
  CUtensorMap tmap;
  {
    cuuint64_t dims[2] = {128, 128};
    cuuint64_t strides[1] = {128 * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("tensor map encode failed %d\n", (int)r);
      return 1;
    }
  }
  size_t smem = sizeof(SemSmem) + 1024;
  CK(cudaFuncSetAttribute(sem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int variant = 0; variant < 2; ++variant) {
  printf("MN-major variant %d (%s)\n", variant, variant == 0 ? "LBO=MN-group stride, SBO=K-group" : "LBO=K-group, SBO=MN-group stride");
  sem_kernel<<<1, 128, smem>>>(tmap, dW1, dW2, dX, dout, variant);
  CK(cudaDeviceSynchronize());
  std::vector<float> out(4 * 128 * kN);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  // references: P(i1, n) = sum_c X(i1,c) W1(c,n); Q(c, n) = sum_i1 X(i1,c) W2(i1,n)
  const char* names[4] = {"SS P (A MN-major)", "SS Q (A K-major)", "TS P (A in TMEM)", "TS Q (A in TMEM)"};
  for (int o = 0; o < 4; ++o) {
    double e_exact = 0, e_tr = 0, e_rn = 0, nrm = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < kN; ++n) {
        double ex = 0, tr = 0, rn = 0;
        for (int k = 0; k < 128; ++k) {
          float a = (o % 2 == 0) ? X[k * 128 + m] : X[m * 128 + k];
          float b = (o % 2 == 0) ? W1[k * kN + n] : W2[k * kN + n];
          ex += (double)a * b;
          tr += (double)tf32_trunc(a) * tf32_trunc(b);
          rn += (double)tf32_rn(a) * tf32_rn(b);
        }
        double g = out[o * 128 * kN + m * kN + n];
        e_exact = fmax(e_exact, fabs(g - ex));
        e_tr = fmax(e_tr, fabs(g - tr));
        e_rn = fmax(e_rn, fabs(g - rn));
        nrm = fmax(nrm, fabs(ex));
      }
    printf("%-20s max|err| vs fp64-exact %.3e, vs trunc-tf32 %.3e, vs rn-tf32 %.3e (max|ref| %.2f)\n",
           names[o], e_exact, e_tr, e_rn, nrm);
  }
  }
  // ---------------- throughput
  const int nsm = prop.multiProcessorCount;
  run_chunk<3, 0>("chunked, commits, no waits", nsm);
  run_chunk<3, 1>("chunked, commit + wait NC back", nsm);
  run_chunk<2, 1>("chunked, commit + wait NC back", nsm);
  run_chunk<6, 1>("chunked, commit + wait NC back", nsm);
  run_tp<2, 48, 0>("TS single", nsm);
  run_tp<6, 48, 0>("TS kernel-mix (A@256)", nsm);
  run_tp<7, 48, 0>("TS kernel-mix (kernel TMEM)", nsm);
  run_tp<8, 48, 0>("TS kernel-mix 1 GEMM", nsm);
  return 0;
  run_tp<0, 80, 0>("SS Kmaj", nsm);
  run_tp<0, 128, 0>("SS Kmaj", nsm);
  run_tp<2, 16, 0>("TS", nsm);
  run_tp<2, 32, 0>("TS", nsm);
  run_tp<2, 48, 0>("TS", nsm);
  run_tp<2, 64, 0>("TS", nsm);
  run_tp<2, 80, 0>("TS", nsm);
  run_tp<2, 96, 0>("TS", nsm);
  run_tp<2, 112, 0>("TS", nsm);
  run_tp<2, 128, 0>("TS", nsm);
  run_tp<3, 48, 0>("TS alt N/N80 (avg)", nsm);
  run_tp<4, 48, 0>("f16 SS Kmaj K=16", nsm);
  run_tp<4, 80, 0>("f16 SS Kmaj K=16", nsm);
  run_tp<5, 48, 0>("f16 TS K=16", nsm);
  run_tp<5, 80, 0>("f16 TS K=16", nsm);
  run_tp<5, 128, 0>("f16 TS K=16", nsm);
  run_tmem_bw(nsm);
  return 0;
}
