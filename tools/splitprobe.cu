// splitprobe.cu — the fused sketch's "split" stage in isolation: 4 warps (one per TMEM lane quarter)
// read a 128x128 SWIZZLE_128B fp32 tile from shared memory in both orientations, split x = hi + lo
// (tf32) and store hi/lo to TMEM.  Reports cycles per 32-column chunk for code variants.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o splitprobe splitprobe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"
using namespace sm100;

__device__ __forceinline__ uint32_t hb(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

template <int VAR, int NW>
__global__ void __launch_bounds__(NW * 32, 1) split_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) float X[];  // 16384 floats
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tslot);
  for (int i = threadIdx.x; i < 16384; i += NW * 32) X[i] = 1.0f + i * 1e-3f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t sub = warp & 3, par = warp >> 2;
  const uint32_t ch0 = tslot + ((32u * sub) << 16);
  const int gq = 32 * sub + lane;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int kc = 0; kc < 4; ++kc) {
      if (NW == 8 && (kc & 1) != (int)par) continue;
      const uint32_t ch = ch0 + (kc & 1) * 128;
#pragma unroll 1
      for (int h0 = 0; h0 < 32; h0 += 16) {
        if (VAR != 2) {  // P layout
          const float* box = X + sub * 4096;
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int g = kc * 32 + h0 + j;
            const float x = box[g * 32 + ((((lane >> 2) ^ (g & 7))) << 2) + (lane & 3)];
            hi[j] = __float_as_uint(x);
            lo[j] = __float_as_uint(x - __uint_as_float(hb(x)));
          }
          tmem_st16(ch + h0, hi);
          tmem_st16(ch + 32 + h0, lo);
        }
        if (VAR != 1) {  // Q layout
          const int rho0 = kc * 32 + h0;
          const float* row = X + (rho0 >> 5) * 4096 + gq * 32;
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int chunk = (((rho0 & 31) >> 2) + qq) ^ (gq & 7);
            const float4 v = *reinterpret_cast<const float4*>(row + chunk * 4);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              hi[qq * 4 + e] = __float_as_uint(vv[e]);
              lo[qq * 4 + e] = __float_as_uint(vv[e] - __uint_as_float(hb(vv[e])));
            }
          }
          tmem_st16(ch + 64 + h0, hi);
          tmem_st16(ch + 96 + h0, lo);
        }
      }
      tmem_st_wait();
    }
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * NW + warp] = (t1 - t0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}

template <int VAR, int NW>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * NW * 8);
  auto k = split_kernel<VAR, NW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  k<<<148, NW * 32, 65536 + 1024>>>(10, d);
  cudaDeviceSynchronize();
  const int iters = 200;
  k<<<148, NW * 32, 65536 + 1024>>>(iters, d);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(148 * NW);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  printf("%-28s warps=%d: %.0f cycles per 128x128 tile (%.0f per 32-col chunk)\n", name, NW,
         h[0] / (double)iters, h[0] / (double)iters / 4);
  cudaFree(d);
}

int main() {
  run<0, 4>("P+Q layouts");
  run<1, 4>("P layout only");
  run<2, 4>("Q layout only");
  run<0, 8>("P+Q layouts, 2 warps/quarter");
  return 0;
}
