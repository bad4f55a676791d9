// krp_common.cuh — shared host/device definitions of libkrp (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/krp.h"

namespace krp {

constexpr int kMaxD = 8;
constexpr int kMaxR = 256;      // sketch width R; rhosvd / sthosvd: R <= kMaxRDecomp
constexpr int kMaxRDecomp = 64; // the fp64 Gram / Cholesky / Jacobi kernels hold R x R in one CTA

// Tensor geometry, first-index-fastest.
struct Dims {
  int d = 0;
  int64_t n[kMaxD] = {};
  int64_t stride[kMaxD] = {};  // stride[k] = prod_{m<k} n[m]
  int64_t N = 0;
};

inline Dims make_dims(int d, const int64_t* dims) {
  Dims g;
  g.d = d;
  int64_t s = 1;
  for (int k = 0; k < d; ++k) {
    g.n[k] = dims[k];
    g.stride[k] = s;
    s *= dims[k];
  }
  g.N = s;
  return g;
}

// Device-pointer table passed by value to kernels.
struct OmegaPtrs {
  const float* p[kMaxD];
};

// Thread-local last error message (krp_last_error_message).
void set_error(const char* fmt, ...);
const char* last_error();

// Launch counter (krp_launch_count).
void count_launch(int n = 1);

// Kernel profiling (krp_profile_*): prof_begin/prof_end bracket one launch of the dominant kernel.
bool prof_on();
void prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s, double alg_bytes, double alg_flops);

#define KRP_CHECK_CUDA(expr)                                                        \
  do {                                                                              \
    cudaError_t e__ = (expr);                                                       \
    if (e__ != cudaSuccess) {                                                       \
      ::krp::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e__),     \
                       __FILE__, __LINE__);                                         \
      return KRP_ECUDA;                                                             \
    }                                                                               \
  } while (0)

#define KRP_CHECK_LAUNCH()                                                          \
  do {                                                                              \
    ::krp::count_launch();                                                          \
    cudaError_t e__ = cudaGetLastError();                                           \
    if (e__ != cudaSuccess) {                                                       \
      ::krp::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(e__), \
                       __FILE__, __LINE__);                                         \
      return KRP_ECUDA;                                                             \
    }                                                                               \
  } while (0)

// Programmatic dependent launch: the kernel may be scheduled while its predecessor in the stream is
// still running; it must call pdl_wait() before touching anything the predecessor writes.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#define KRP_TRY(expr)              \
  do {                             \
    int s__ = (expr);              \
    if (s__ != KRP_OK) return s__; \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over the caller's workspace (256-byte aligned pieces).
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  bool measuring = false;  // when true only sizes are accumulated
  template <class T>
  T* take(size_t count) {
    size_t bytes = align_up(count * sizeof(T), 256);
    T* p = measuring ? nullptr : reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
  bool overflow() const { return !measuring && off > cap; }
};

}  // namespace krp
