// splitbench.cu — micro-benchmark of the sketch kernel's split stage (dev tool): 4 warps read a
// 128x128 fp32 SWIZZLE_128B tile from shared memory in the P view (lane = ρ, scalar loads) and the Q
// view (lane = γ, 16-byte loads), form lo = x - tf32(x), and store P-hi, P-lo, Q-lo to TMEM in
// 32-column chunks.  Variants isolate the cost of each part (cycles per 32-column chunk per warp).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o splitbench splitbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"

using namespace sm100;

__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t hib(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

template <int VAR, int BG = 0>
__global__ void __launch_bounds__(160, 1) split_kernel(int iters, unsigned long long* out, float* sink,
                                                       const float* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tb_s;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* xs = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < 16384; i += 128) xs[i] = 1.0f + i * 1e-3f;
  __shared__ uint64_t lb[2];
  if (warp == 0) tmem_alloc<512>(&tb_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  __shared__ uint64_t hs_full[2], hs_ready[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&hs_full[i], 4);
      mbar_init(&hs_ready[i], 1);
    }
    fence_barrier_init();
  }
  asm volatile("bar.sync 2, 160;");
  if (warp == 4 && VAR == 4) {  // partner: waits full[c], arrives ready[c] (like the MMA warp's commit)
    for (int c = 0; c < iters * 4; ++c) {
      mbar_wait(&hs_full[c & 1], (c >> 1) & 1);
      if (elect_one()) mbar_arrive(&hs_ready[c & 1]);
      __syncwarp();
    }
    return;
  }
  if (warp == 4) {  // background bulk copies into a second 64 KB region (TMA-like SMEM writes)
    if (BG && elect_one()) {
      float* land = xs + 16384;
      mbar_init(&lb[0], 1);
      mbar_init(&lb[1], 1);
      fence_barrier_init();
      uint32_t ph[2] = {0, 0};
      for (int i = 0; i < 2; ++i) {
        mbar_arrive_expect_tx(&lb[i], 32768);
        bulk_copy_g2s(land + i * 8192, gsrc + (size_t)(blockIdx.x * 64 + i) * 8192, 32768, &lb[i]);
      }
      for (int i = 2; i < iters * 2; ++i) {
        const int b = i & 1;
        mbar_wait(&lb[b], ph[b]);
        ph[b] ^= 1;
        mbar_arrive_expect_tx(&lb[b], 32768);
        bulk_copy_g2s(land + b * 8192, gsrc + ((size_t)(blockIdx.x * 997 + i) % 32768) * 8192, 32768, &lb[b]);
      }
      mbar_wait(&lb[0], ph[0]);
      mbar_wait(&lb[1], ph[1]);
    }
    return;
  }
  const uint32_t sub = warp;
  const uint32_t ch0 = tb_s + ((32u * sub) << 16);
  uint32_t psw[8];
  for (int j = 0; j < 8; ++j)
    psw[j] = smem_u32(xs) + sub * 16384u + ((((lane >> 2) ^ static_cast<uint32_t>(j)) << 4) | ((lane & 3u) << 2));
  const uint32_t gq = 32 * sub + lane;
  const uint32_t qrow = smem_u32(xs) + gq * 128u, qx = gq & 7;
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int kc = 0; kc < 4; ++kc) {
      const int c = it * 4 + kc;
      if (VAR == 4 && c >= 2) {
        mbar_wait(&hs_ready[c & 1], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      const uint32_t ch = ch0 + (kc & 1) * 96;
      uint32_t px[32];
      float qv[32];
      const uint32_t goff = kc * 32 * 128u;
      if (VAR != 3) {
#pragma unroll
        for (int j = 0; j < 32; ++j) px[j] = __float_as_uint(lds_f32(psw[j & 7] + goff + j * 128u));
        const uint32_t rowa = qrow + kc * 16384u;
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) lds_v4(rowa + (((uint32_t)qq ^ qx) << 4), qv[4 * qq], qv[4 * qq + 1], qv[4 * qq + 2], qv[4 * qq + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) px[j] = __float_as_uint(1.0f + j + it), qv[j] = 2.0f + j + kc;
      }
      uint32_t lo[32], ql[32];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        float2 l = f2_sub(make_float2(__uint_as_float(px[j]), __uint_as_float(px[j + 1])),
                          make_float2(__uint_as_float(hib(__uint_as_float(px[j]))), __uint_as_float(hib(__uint_as_float(px[j + 1])))));
        lo[j] = __float_as_uint(l.x);
        lo[j + 1] = __float_as_uint(l.y);
        float2 m = f2_sub(make_float2(qv[j], qv[j + 1]), make_float2(__uint_as_float(hib(qv[j])), __uint_as_float(hib(qv[j + 1]))));
        ql[j] = __float_as_uint(m.x);
        ql[j + 1] = __float_as_uint(m.y);
      }
      if (VAR == 0 || VAR == 2 || VAR == 3 || VAR == 4) {
        tmem_st32(ch, px);
        tmem_st32(ch + 32, lo);
        tmem_st32(ch + 64, ql);
        if (VAR != 2) tmem_st_wait();
        if (VAR == 4) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&hs_full[c & 1]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += __uint_as_float(px[j] ^ lo[j] ^ ql[j]);
      }
    }
  }
  if (VAR == 2) tmem_st_wait();
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 4 + warp] = t1 - t0;
  sink[blockIdx.x * 128 + threadIdx.x] = acc;
  tc_fence_before();
  asm volatile("bar.sync 1, 128;");
  if (warp == 0) tmem_dealloc<512>(tb_s);
}

template <int VAR, int BG = 0>
void run(const char* name, int nsm) {
  static float* gsrc = nullptr;
  if (!gsrc) cudaMalloc(&gsrc, (size_t)32768 * 8192 * 4);
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, nsm * 4 * 8);
  cudaMalloc(&sink, nsm * 128 * 4);
  cudaFuncSetAttribute(split_kernel<VAR, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  const int iters = 2000;
  split_kernel<VAR, BG><<<nsm, 160, 140000>>>(10, d, sink, gsrc);
  split_kernel<VAR, BG><<<nsm, 160, 140000>>>(iters, d, sink, gsrc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(nsm * 4);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  double m = 0;
  for (auto v : h) m = v > m ? v : m;
  printf("%-40s %8.1f cycles per 32-col chunk per warp (%s)\n", name, m / (iters * 4.0), cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  int nsm = 148;
  run<0>("full: LDS + split + 3x STTM.x32 + wait", nsm);
  run<4>("full + fences + mbarrier handshake (NC=2)", nsm);
  run<0, 1>("full + background bulk copies (TMA-like)", nsm);
  run<1, 1>("no TMEM store + background bulk copies", nsm);
  run<1>("no TMEM store", nsm);
  run<2>("STTM without per-chunk wait", nsm);
  run<3>("no LDS (register data) + STTM + wait", nsm);
  return 0;
}
