// pipebench.cu — the sketch kernel's split -> MMA chunk pipeline without data (dev tool).
// Warps 0-3 ("split") wait chunk_empty[c % NC], optionally write 3 x 32 TMEM columns (P hi, P lo, Q lo)
// for their lane quarter, and arrive on chunk_full; the MMA warp(s) wait chunk_full, issue the chunk's
// MMAs (P: TS N=80 + TS N=48; Q: SS N=80 + TS N=48; 4 K-steps) and commit to chunk_empty.
// Reports cycles per 32-column chunk.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o pipebench pipebench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"

using namespace sm100;

struct alignas(1024) Smem {
  float a[4][128][32];
  float b[2][4][80][32];
  uint64_t full[4], empty[4], fullx[2], emptyx[2], accf[2];
  float wsb[2][64];
  uint32_t tbase;
};

// STORE: split warps write TMEM; ISSUERS: 1 (one warp issues P and Q) or 2 (P warp, Q warp); NC stages
// TILE: 1 = per-tile stage handshake with a producer warp (full_x / empty_x, NS = 2, the Q issuer commits
// to empty_x); 2 = plus a per-tile acc_full commit and an Ω_S bulk copy (as in the sketch kernel)
template <int STORE, int ISSUERS, int NC, int TILE = 0>
__global__ void __launch_bounds__(224, 1) pipe_kernel(int chunks, unsigned long long* out, const float* oms) {
  extern __shared__ __align__(1024) uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * 128 * 32; i += blockDim.x) (&s.a[0][0][0])[i] = 1.0f;
  for (int i = threadIdx.x; i < 2 * 4 * 80 * 32; i += blockDim.x) (&s.b[0][0][0][0])[i] = 0.5f;
  if (warp == 4) tmem_alloc<512>(&s.tbase);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NC; ++i) {
      mbar_init(&s.full[i], 4);
      mbar_init(&s.empty[i], ISSUERS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.fullx[i], 1);
      mbar_init(&s.emptyx[i], TILE == 3 ? 4 : 4 + 1);
      mbar_init(&s.accf[i], ISSUERS + 1);
    }
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = s.tbase;
  long long t0 = clock64();
  if (warp < 4) {
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(1.0f + j);
    for (int c = 0; c < chunks; ++c) {
      const int st = c % NC;
      const int t = c >> 2;
      if (TILE && (c & 3) == 0) mbar_wait(&s.fullx[t & 1], (t >> 1) & 1);
      mbar_wait(&s.empty[st], ((c / NC) & 1) ^ 1);
      tc_fence_after();
      if (STORE) {
        const uint32_t ch = tb + ((32u * warp) << 16) + 320 + st * 96;
        tmem_st32(ch, v);
        tmem_st32(ch + 32, v);
        tmem_st32(ch + 64, v);
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.full[st]);
      if (TILE && (c & 3) == 3 && lane == 0) mbar_arrive(&s.emptyx[t & 1]);
    }
  } else if (TILE && warp == 6) {  // producer: waits the stage free, marks it full (no data)
    if (elect_one()) {
      for (int t = 0; t < chunks / 4; ++t) {
        if (t >= 2) {
          mbar_wait(&s.emptyx[t & 1], ((t >> 1) - 1) & 1);
          if (TILE == 3) mbar_wait(&s.accf[t & 1], ((t >> 1) - 1) & 1);
        }
        mbar_arrive(&s.fullx[t & 1]);
      }
    }
  } else if (warp == 4 || (ISSUERS == 2 && warp == 5)) {
    const bool leader = elect_one();
    const bool doP = ISSUERS == 1 || warp == 4, doQ = ISSUERS == 1 || warp == 5;
    const uint32_t idc = make_idesc_tf32(128, 80, 0, 0), idl = make_idesc_tf32(128, 48, 0, 0);
    const uint64_t bp0 = make_smem_desc(smem_u32(&s.b[0][0][0][0]), 0, 1024, kLayoutSW128);
    const uint64_t bq0 = make_smem_desc(smem_u32(&s.b[1][0][0][0]), 0, 1024, kLayoutSW128);
    const uint64_t a0 = make_smem_desc(smem_u32(&s.a[0][0][0]), 0, 1024, kLayoutSW128);
    for (int c = 0; c < chunks; ++c) {
      const int st = c % NC;
      const int t = c >> 2;
      if (TILE >= 2 && (c & 3) == 0 && doP && leader) {
        mbar_arrive_expect_tx(&s.accf[t & 1], 256);
        bulk_copy_g2s(&s.wsb[t & 1][0], oms + (t & 511) * 64, 256, &s.accf[t & 1]);
      }
      mbar_wait(&s.full[st], (c / NC) & 1);
      tc_fence_after();
      const uint32_t ach = tb + 320 + st * 96;
      const int kk0 = (c & 3) * 4;
      if (leader) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t koff = (kk0 >> 2) * (80 * 8) + ks * 2;
          const uint32_t acc = (kk0 + ks) > 0 ? 1u : 0u;
          if (doP) {
            mma_tf32_ts(tb + 0, ach + 8 * ks, bp0 + koff, idc, acc);
            mma_tf32_ts(tb + 0, ach + 32 + 8 * ks, bp0 + koff, idl, 1u);
          }
          if (doQ) {
            mma_tf32_ss(tb + 80, a0 + (kk0 >> 2) * 1024 + ks * 2, bq0 + koff, idc, acc);
            mma_tf32_ts(tb + 80, ach + 64 + 8 * ks, bq0 + koff, idl, 1u);
          }
        }
        mma_commit(&s.empty[st]);
        if ((TILE == 1 || TILE == 2) && (c & 3) == 3 && doQ) mma_commit(&s.emptyx[t & 1]);
        if (TILE >= 2 && (c & 3) == 3) mma_commit(&s.accf[t & 1]);
      }
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc<512>(tb);
}

template <int STORE, int ISSUERS, int NC, int TILE = 0>
void run(const char* name) {
  const int nsm = 148, chunks = 20000;
  auto k = pipe_kernel<STORE, ISSUERS, NC, TILE>;
  static float* oms = nullptr;
  if (!oms) cudaMalloc(&oms, 512 * 64 * 4);
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  k<<<nsm, 224, smem>>>(100, d, oms);
  k<<<nsm, 224, smem>>>(chunks, d, oms);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(nsm);
  cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  printf("%-48s NC=%d: %7.1f cyc/chunk (%s)\n", name, NC, mx / chunks, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<1, 2, 2>("split TMEM stores, 2 issuers");
  run<1, 2, 2, 2>("  + tile handshake, acc_full commit, bulk copy");
  run<1, 2, 2, 3>("  same, stage released through acc_full");
  run<1, 1, 2>("split TMEM stores, 1 issuer");
  run<1, 1, 2, 2>("  + tile handshake, acc_full commit, bulk copy");
  run<1, 1, 2, 3>("  same, stage released through acc_full");
  run<1, 1, 3, 3>("  same, NC=3");
  return 0;
}
