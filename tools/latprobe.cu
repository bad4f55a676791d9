// latprobe.cu — latencies that bound the split/epilogue pipelines of the fused sketch:
// tcgen05.st + wait::st, tcgen05.ld + wait::ld (x8/x16/x32), mbarrier ping-pong between warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o latprobe latprobe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"
using namespace sm100;

__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%"
      "29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__global__ void __launch_bounds__(256, 1) lat_kernel(int nwarps_active, int mode, unsigned long long* out) {
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar[2];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot + (((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = lane + i;
  const int iters = 1000;
  long long t0 = 0, t1 = 0;
  float acc = 0.f;
  if (mode < 6 && static_cast<int>(warp) < nwarps_active) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode == 0) {
        tmem_st8(tb, r);
        tmem_st_wait();
      } else if (mode == 1) {
        tmem_st16(tb, r);
        tmem_st_wait();
      } else if (mode == 2) {
        st32(tb, r);
        tmem_st_wait();
      } else if (mode == 3) {
        float v[8];
        tmem_ld8(tb, v);
        tmem_ld_wait();
        acc += v[0];
      } else if (mode == 4) {
        float v[16];
        tmem_ld16(tb, v);
        tmem_ld_wait();
        acc += v[0];
      } else {  // 4 x st16 then one wait
        tmem_st16(tb, r);
        tmem_st16(tb + 16, r);
        tmem_st16(tb + 32, r);
        tmem_st16(tb + 48, r);
        tmem_st_wait();
      }
    }
    t1 = clock64();
  } else if (mode == 6 && warp < 2) {
    // mbarrier ping-pong: warp 0 arrives on bar[0], warp 1 waits then arrives on bar[1]
    t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (warp == 0) {
        if (lane == 0) mbar_arrive(&bar[0]);
        mbar_wait(&bar[1], ph);
      } else {
        mbar_wait(&bar[0], ph);
        if (lane == 0) mbar_arrive(&bar[1]);
      }
      ph ^= 1;
    }
    t1 = clock64();
  }
  if (lane == 0 && warp < 8) out[blockIdx.x * 8 + warp] = (t1 - t0) / iters + (acc == 12345.f);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8 * 8);
  const char* names[7] = {"st.x8+wait", "st.x16+wait", "st.x32+wait", "ld.x8+wait", "ld.x16+wait",
                          "4x st.x16 + 1 wait", "mbarrier ping-pong (round trip)"};
  for (int mode = 0; mode < 7; ++mode) {
    for (int nw : {1, 4, 8}) {
      if (mode == 6 && nw != 1) continue;
      lat_kernel<<<148, 256>>>(nw, mode, d);
      cudaDeviceSynchronize();
      std::vector<unsigned long long> h(148 * 8);
      cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
      printf("%-32s warps=%d : %llu cycles/iter (warp0 of CTA0)\n", names[mode], nw, h[0]);
    }
  }
  return 0;
}
