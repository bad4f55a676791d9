// tmaprobe.cu — HBM->SMEM streaming rate of TMA box shapes for a 128x128 fp32 tile
// (the fused sketch's tile), 1 persistent CTA per SM, no consumers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmaprobe tmaprobe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
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

struct Cfg {
  int mode;      // 0: 3D box {32,128,1} x4 ; 1: 2D box {32,128} x4 ; 2: 2D box {128,32} x4 (no swizzle)
                 // 3: 1D bulk copies 128 x 512 B ; 4: 2D box {32,256} x 2 half-tiles? (32 rows of 2 tiles)
  int stages;    // stages of 64 KB
  int64_t M, C, S;
};

__global__ void __launch_bounds__(128, 1) tma_kernel(const __grid_constant__ CUtensorMap tmap, const float* X,
                                                     Cfg cfg, int64_t T, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + cfg.stages * 65536);
  if (threadIdx.x == 0) {
    for (int i = 0; i < cfg.stages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t t0 = blockIdx.x * T / gridDim.x, t1 = (blockIdx.x + 1) * T / gridDim.x;
  const int64_t RB = cfg.M / 128, CB = cfg.C / 128;
  long long c0 = clock64();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    int st = 0;
    uint32_t ph = 0;
    int64_t issued = t0, done = t0;
    // keep `stages` tiles in flight
    while (done < t1) {
      while (issued < t1 && issued - done < cfg.stages) {
        const int s_ = static_cast<int>((issued - t0) % cfg.stages);
        const int64_t pair = issued / cfg.S, s = issued % cfg.S;
        const int rb = pair / CB, cb = pair % CB;
        mbar_arrive_expect_tx(&full[s_], 65536);
        uint8_t* dst = sm + s_ * 65536;
        if (cfg.mode == 0) {
          for (int j = 0; j < 4; ++j) tma_load_3d(dst + j * 16384, &tmap, &full[s_], rb * 128 + 32 * j, cb * 128, s, pol);
        } else if (cfg.mode == 1) {
          for (int j = 0; j < 4; ++j)
            tma_load_2d(dst + j * 16384, &tmap, &full[s_], rb * 128 + 32 * j, static_cast<int>(cb * 128 + s * cfg.C), pol);
        } else if (cfg.mode == 2) {
          for (int j = 0; j < 4; ++j)
            tma_load_2d(dst + j * 16384, &tmap, &full[s_], rb * 128, static_cast<int>(cb * 128 + 32 * j + s * cfg.C), pol);
        } else if (cfg.mode == 3) {
          for (int g = 0; g < 128; ++g) {
            const float* src = X + (rb * 128) + cfg.M * (cb * 128 + g + cfg.C * s);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                    smem_u32(dst + g * 512)),
                "l"(src), "r"(512), "r"(smem_u32(&full[s_])), "l"(pol)
                : "memory");
          }
        }
        ++issued;
      }
      const int s_ = static_cast<int>((done - t0) % cfg.stages);
      const uint32_t par = static_cast<uint32_t>(((done - t0) / cfg.stages) & 1);
      mbar_wait(&full[s_], par);
      ++done;
    }
    cyc[blockIdx.x] = clock64() - c0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int main() {
  const int64_t M = 512, C = 512, S = 512;
  const size_t N = M * C * S;
  float* X;
  CK(cudaMalloc(&X, N * 4));
  CK(cudaMemset(X, 0, N * 4));
  int nsm = 148;
  unsigned long long* cyc;
  CK(cudaMalloc(&cyc, nsm * 8));
  const int64_t T = (M / 128) * (C / 128) * S;
  for (int mode = 0; mode < 4; ++mode) {
    for (int stages : {2, 3}) {
      CUtensorMap tm;
      CUresult r;
      if (mode == 0) {
        cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)C, (cuuint64_t)S};
        cuuint64_t str[2] = {(cuuint64_t)M * 4, (cuuint64_t)M * C * 4};
        cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
        r = enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)(C * S)};
        cuuint64_t str[1] = {(cuuint64_t)M * 4};
        cuuint32_t box1[2] = {32, 128}, box2[2] = {128, 32}, es[2] = {1, 1};
        r = enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, mode == 2 ? box2 : box1, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, mode == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (r != CUDA_SUCCESS) {
        printf("encode failed mode %d\n", mode);
        continue;
      }
      Cfg cfg{mode, stages, M, C, S};
      size_t smem = stages * 65536 + 1024 + 256;
      CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      tma_kernel<<<nsm, 128, smem>>>(tm, X, cfg, T, cyc);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) tma_kernel<<<nsm, 128, smem>>>(tm, X, cfg, T, cyc);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("mode %d stages %d: %.1f us  %.0f GB/s\n", mode, stages, ms * 1e3, N * 4.0 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
