// latbench.cu — handshake latencies inside one CTA (dev tool):
//  (1) mbarrier ping-pong between two warps (arrive -> try_wait) with and without a suspend-time hint
//  (2) the sketch kernel's chunk round trip without work: 4 "split" warps arrive on full[c], one "MMA"
//      thread waits, issues tcgen05.commit (no MMAs outstanding) to empty[c], the split warps wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o latbench latbench.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"

using namespace sm100;

__device__ __forceinline__ void wait_spin(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

template <int HINT>
__device__ __forceinline__ void wait_any(uint64_t* bar, uint32_t parity) {
  if (HINT) mbar_wait(bar, parity);
  else wait_spin(bar, parity);
}

template <int HINT>
__global__ void pingpong(int iters, long long* out) {
  __shared__ uint64_t bars[2];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (warp == 0) {
      if ((threadIdx.x & 31) == 0) mbar_arrive(&bars[0]);
      wait_any<HINT>(&bars[1], i & 1);
    } else if (warp == 1) {
      wait_any<HINT>(&bars[0], i & 1);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&bars[1]);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// chunk round trip: NC stages; split warps 0-3, MMA warp 4
template <int HINT, int NC>
__global__ void roundtrip(int iters, long long* out) {
  __shared__ uint64_t full[8], empty[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 4) tmem_alloc<32>(&tslot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NC; ++i) {
      mbar_init(&full[i], 4);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long t0 = clock64();
  if (warp < 4) {
    for (int c = 0; c < iters; ++c) {
      const int st = c % NC;
      wait_any<HINT>(&empty[st], ((c / NC) & 1) ^ 1);
      tc_fence_after();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&full[st]);
    }
  } else if (warp == 4) {
    const bool leader = elect_one();
    for (int c = 0; c < iters; ++c) {
      const int st = c % NC;
      wait_any<HINT>(&full[st], (c / NC) & 1);
      tc_fence_after();
      if (leader) mma_commit(&empty[st]);
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc<32>(tslot);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  long long h;
  const int it = 20000;
  pingpong<0><<<148, 64>>>(it, d);
  pingpong<0><<<148, 64>>>(it, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mbarrier ping-pong, spin try_wait      : %.1f cycles per one-way handoff\n", h / (2.0 * it));
  pingpong<1><<<148, 64>>>(it, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mbarrier ping-pong, suspend-hint wait  : %.1f cycles per one-way handoff\n", h / (2.0 * it));
  roundtrip<0, 1><<<148, 160>>>(it, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("chunk round trip (4 arrive -> commit), NC=1, spin : %.1f cycles per chunk\n", h / (1.0 * it));
  roundtrip<1, 1><<<148, 160>>>(it, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("chunk round trip (4 arrive -> commit), NC=1, hint : %.1f cycles per chunk\n", h / (1.0 * it));
  roundtrip<1, 2><<<148, 160>>>(it, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("chunk round trip (4 arrive -> commit), NC=2, hint : %.1f cycles per chunk\n", h / (1.0 * it));
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
