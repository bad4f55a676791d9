// mmabench.cu — tensor-core throughput of the sketch kernel's per-chunk MMA mix (dev tool).
// One chunk = 4 K-steps (K = 8 each) of the two GEMMs at M = 128:
//   P: A from TMEM, hi x [B_hi | B_lo] (N = NC) + lo x B_hi (N = NL)
//   Q: A_hi from SMEM (SS, K-major SW128) or TMEM, hi x [B_hi | B_lo] + lo (TMEM) x B_hi
// Variants: one or two issuing threads, Q-hi from SMEM or TMEM, commit per chunk.  Reports cycles per
// chunk (all SMs busy, so the clock is the loaded one).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mmabench mmabench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"

using namespace sm100;

struct alignas(1024) Smem {
  float a[4][128][32];  // 64 KB tile, 4 boxes {32 K, 128 rows}, SW128 K-major
  float land[2][4096];  // 2 x 16 KB landing buffers for the background bulk copies (BG variants)
  float b[2][4][96][32];  // two B images (P, Q): 4 K atoms x up to 96 rows x 32
  uint64_t bar[8];
  uint32_t tbase;
};

// VAR: 0 = one issuer, Q-hi SS; 1 = one issuer, Q-hi TS; 2 = two issuers (P / Q warps), Q-hi SS;
//      3 = P only (TS); 4 = Q only (SS hi); 5 = one issuer, all TS, N=NC only (no lo x hi)
template <int VAR, int NCAT, int NLO, int BG = 0, int RND = 0>
__global__ void __launch_bounds__(128, 1) mma_kernel(int chunks, unsigned long long* out, const float* gsrc = nullptr,
                                                     volatile int* stop = nullptr) {
  extern __shared__ __align__(1024) uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4 * 128 * 32; i += 128)
    (&s.a[0][0][0])[i] = RND ? __uint_as_float(0x3f800000u | ((i * 2654435761u) >> 9)) * ((i & 1) ? 1.f : -1.f) : 1.0f;
  for (int i = threadIdx.x; i < 2 * 4 * 96 * 32; i += 128)
    (&s.b[0][0][0][0])[i] = RND ? __uint_as_float(0x3f000000u | ((i * 40503u * 2654435761u) >> 9)) * ((i & 2) ? 1.f : -1.f) : 0.5f;
  if (warp == 0) tmem_alloc<512>(&s.tbase);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&s.bar[i], VAR == 2 ? 2 : 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = s.tbase;
  const uint32_t idc = make_idesc_tf32(128, NCAT, 0, 0), idl = make_idesc_tf32(128, NLO, 0, 0);
  const uint64_t bp0 = make_smem_desc(smem_u32(&s.b[0][0][0][0]), 0, 1024, kLayoutSW128);
  const uint64_t bq0 = make_smem_desc(smem_u32(&s.b[1][0][0][0]), 0, 1024, kLayoutSW128);
  const uint64_t a0 = make_smem_desc(smem_u32(&s.a[0][0][0]), 0, 1024, kLayoutSW128);
  const uint64_t katom = 96 * 8;
  const bool issuer = (VAR == 2) ? (warp < 2) : (warp == 0);
  if (BG && warp == 3) {  // background producer: 16 KB bulk copies global -> SMEM, as fast as they land
    if (elect_one()) {
      __shared__ uint64_t lb[2];
      mbar_init(&lb[0], 1);
      mbar_init(&lb[1], 1);
      fence_barrier_init();
      uint32_t ph[2] = {0, 0};
      for (int i = 0; i < 2; ++i) {
        mbar_arrive_expect_tx(&lb[i], 16384);
        bulk_copy_g2s(&s.land[i][0], gsrc + (size_t)(blockIdx.x * 64 + i) * 4096, 16384, &lb[i]);
      }
      for (int i = 2; i < chunks * 3 / 4 + 2; ++i) {  // ~ 12 KB per chunk (64 KB per 4 chunks + margin)
        const int b = i & 1;
        mbar_wait(&lb[b], ph[b]);
        ph[b] ^= 1;
        mbar_arrive_expect_tx(&lb[b], 16384);
        bulk_copy_g2s(&s.land[b][0], gsrc + ((size_t)(blockIdx.x * 997 + i) % 65536) * 4096, 16384, &lb[b]);
      }
      mbar_wait(&lb[0], ph[0]);
      mbar_wait(&lb[1], ph[1]);
    }
  }
  long long t0 = clock64();
  if (issuer && elect_one()) {
    const bool doP = VAR != 4 && !(VAR == 2 && warp == 1);
    const bool doQ = VAR != 3 && !(VAR == 2 && warp == 0);
    for (int c = 0; c < chunks; ++c) {
      const int st = c & 1;
      if (c >= 2) mbar_wait(&s.bar[st], ((c >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t dP = tb + 0, dQ = tb + 96;
      const uint32_t ach = tb + 192 + st * 128;  // P hi, P lo, Q hi, Q lo: 32 cols each
      const int kk0 = (c & 3) * 4;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t koff = (kk0 >> 2) * katom + ks * 2;
        const uint32_t acc = (kk0 + ks) > 0 ? 1u : 0u;
        if (doP) {
          mma_tf32_ts(dP, ach + 8 * ks, bp0 + koff, idc, acc);
          if (VAR != 5) mma_tf32_ts(dP, ach + 32 + 8 * ks, bp0 + koff, idl, 1u);
        }
        if (doQ) {
          if (VAR == 1 || VAR == 5)
            mma_tf32_ts(dQ, ach + 64 + 8 * ks, bq0 + koff, idc, acc);
          else
            mma_tf32_ss(dQ, a0 + (kk0 >> 2) * 1024 + ks * 2, bq0 + koff, idc, acc);
          if (VAR != 5) mma_tf32_ts(dQ, ach + 96 + 8 * ks, bq0 + koff, idl, 1u);
        }
      }
      mma_commit(&s.bar[st]);
    }
    for (int c = chunks - 2; c < chunks; ++c) mbar_wait(&s.bar[c & 1], (c >> 1) & 1);
  }
  __syncwarp();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int VAR, int NCAT, int NLO, int BG = 0, int RND = 0>
void run(const char* name) {
  const int nsm = 148, chunks = 20000;
  auto k = mma_kernel<VAR, NCAT, NLO, BG, RND>;
  static float* gsrc = nullptr;
  if (!gsrc) cudaMalloc(&gsrc, (size_t)65536 * 4096 * 4);  // 1 GiB source for the background copies
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  k<<<nsm, 128, smem>>>(100, d, gsrc, nullptr);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<nsm, 128, smem>>>(chunks, d, gsrc, nullptr);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(nsm);
  cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  printf("%-44s NCAT=%3d NLO=%3d: %7.1f cyc/chunk  clk %.0f MHz  (%s)\n", name, NCAT, NLO, mx / chunks,
         mx / (ms * 1e-3) / 1e6, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<2, 80, 48>("2 issuers, Q SS-hi, constant data");
  run<2, 80, 48, 0, 1>("2 issuers, Q SS-hi, random data");
  run<1, 80, 48>("1 issuer, Q TS-hi, constant data");
  run<1, 80, 48, 0, 1>("1 issuer, Q TS-hi, random data");
  run<3, 80, 48, 0, 1>("P only, random data");
  return 0;
}
