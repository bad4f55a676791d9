// cpprobe.cu — tcgen05.cp (SMEM -> TMEM) for the Q view of the sketch tile (dev tool).
// (1) correctness: a 128 x 32 fp32 box in the TMA SWIZZLE_128B layout (rows = γ, 128 B = 32 ρ) copied
//     with 4 x tcgen05.cp.128x256b (one per 8-column K-step, same descriptors as the SS A operand) must
//     land as TMEM lane γ, column ρ.
// (2) throughput of the Q-lo path per 32-column chunk: cp (4x) + commit/wait, then each of 4 warps does
//     tcgen05.ld 32x32b.x32, lo = x - tf32(x), tcgen05.st back in place.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o cpprobe cpprobe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2507_23207_b200/csrc/sm100.cuh"

using namespace sm100;

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

struct alignas(1024) Smem {
  float box[4][128][32];
  uint64_t bar[2];
  uint32_t tbase;
};

__global__ void __launch_bounds__(128, 1) cp_kernel(int iters, float* out, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // element (ρ, γ) of box b at byte γ*128 + (((ρ%32)/4 ^ (γ%8)) << 4) + (ρ%4)*4: value = 1000*γ + 32*b + ρ%32
  for (int i = threadIdx.x; i < 4 * 128 * 32; i += 128) {
    const int b = i / 4096, g = (i / 32) % 128, r = i % 32;
    const int off = g * 128 + ((((r >> 2) ^ (g & 7))) << 4) + (r & 3) * 4;
    reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(&s.box[b][0][0]) + off)[0] = 1000.f * g + 32 * b + r;
  }
  if (warp == 0) tmem_alloc<512>(&s.tbase);
  if (threadIdx.x == 0) {
    mbar_init(&s.bar[0], 1);
    mbar_init(&s.bar[1], 4);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = s.tbase;
  const uint64_t d0 = make_smem_desc(smem_u32(&s.box[0][0][0]), 0, 1024, kLayoutSW128);
  // (1) copy all 4 boxes: columns 32b + 8ks + (0..7)
  if (warp == 0 && elect_one()) {
    for (int b = 0; b < 4; ++b)
      for (int ks = 0; ks < 4; ++ks) tmem_cp_128x256b(tb + 32 * b + 8 * ks, d0 + b * 1024 + ks * 2);
    mma_commit(&s.bar[0]);
  }
  mbar_wait(&s.bar[0], 0);
  tc_fence_after();
  {
    const uint32_t ta = tb + ((32u * warp) << 16);
    for (int c = 0; c < 128; c += 16) {
      float v[16];
      tmem_ld16(ta + c, v);
      tmem_ld_wait();
      for (int j = 0; j < 16; ++j) out[(blockIdx.x * 128 + 32 * warp + lane) * 128 + c + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // (2) throughput: per chunk, cp 4 K-steps into cols 128.., then every warp ld -> lo -> st in place
  long long t0 = clock64();
  uint32_t ph0 = 1, ph1 = 0;
  for (int it = 0; it < iters; ++it) {
    const int kc = it & 3;
    if (warp == 0 && elect_one()) {
      if (it > 0) {
        mbar_wait(&s.bar[1], ph1);  // all 4 warps finished the previous chunk
        ph1 ^= 1;
      }
      tc_fence_after();
      for (int ks = 0; ks < 4; ++ks) tmem_cp_128x256b(tb + 128 + 8 * ks, d0 + kc * 1024 + ks * 2);
      mma_commit(&s.bar[0]);
    }
    mbar_wait(&s.bar[0], ph0 & 1);
    ph0 ^= 1;
    tc_fence_after();
    const uint32_t ta = tb + ((32u * warp) << 16) + 128;
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    tmem_ld_wait();
    uint32_t lo[32];
    for (int j = 0; j < 32; j += 2) {
      const float2 l = f2_sub(make_float2(__uint_as_float(v[j]), __uint_as_float(v[j + 1])),
                              make_float2(__uint_as_float(v[j] & 0xFFFFE000u), __uint_as_float(v[j + 1] & 0xFFFFE000u)));
      lo[j] = __float_as_uint(l.x);
      lo[j + 1] = __float_as_uint(l.y);
    }
    tmem_st32(ta, lo);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.bar[1]);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  const int nsm = 148, iters = 4000;
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, (size_t)nsm * 128 * 128 * 4);
  cudaMalloc(&cyc, nsm * 8);
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(cp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cp_kernel<<<nsm, 128, smem>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> h(128 * 128);
  cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int g = 0; g < 128; ++g)
    for (int c = 0; c < 128; ++c) {
      const float want = 1000.f * g + c;  // lane γ, column ρ = 32b + ρ%32
      if (h[g * 128 + c] != want && bad++ < 5) printf("mismatch lane %d col %d: %g vs %g\n", g, c, h[g * 128 + c], want);
    }
  printf("layout check: %s (%d mismatches)\n", bad ? "FAIL" : "ok", bad);
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("Q-lo path (cp 4x128x256b + ld x32 + lo + st x32, 4 warps): %.1f cycles per 32-col chunk\n", (double)c / iters);
  return 0;
}
