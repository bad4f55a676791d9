// krp_baselines.cu — the paper's dense-Gaussian comparison baselines (NEXT-2; Table 1).
//
// RHOSVD / RSTHOSVD sketch each mode with a dense Gaussian test matrix Omega_n in R^{(N/I_n) x l}:
// Y_n = X_(n) Omega_n.  On the first mode X_(1) is X itself (first index fastest); for the others the
// tensor is unfolded explicitly (the paper's "Unfolding" cost, Fig. 3) by a tiled batched transpose, and
// the product is one plain fp32 GEMM (cuBLAS SGEMM, no TF32: library GEMM for a baseline).  These
// are baselines the KRP path is compared against, not the product's hot path.
#include <dlfcn.h>

#include <mutex>

#include "krp_common.cuh"
#include "krp_internal.h"

namespace krp {
namespace {

// U[c][a][i] = X[c][i][a]: mode n moved to be the fastest index, so the unfolding X_(n) is the column-major
// I_n x (N/I_n) matrix U with columns in the order a + A*c (A = prod_{k<n} I_k), i.e. the column order of
// X_(n).  32x32 shared-memory tiles per (c, i-block, a-block).
__global__ void __launch_bounds__(256) unfold_kernel(const float* __restrict__ X, int64_t A, int64_t In, int64_t Cc,
                                                    float* __restrict__ U) {
  __shared__ float tile[32][33];
  const int64_t nbi = (In + 31) / 32, nba = (A + 31) / 32;
  int64_t b = blockIdx.x;
  const int64_t c = b / (nbi * nba);
  b -= c * nbi * nba;
  const int64_t bi = b / nba, ba = b - bi * nba;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const float* src = X + c * In * A;
  float* dst = U + c * In * A;
  for (int k = ty; k < 32; k += 8) {  // read rows i (stride A), a contiguous
    const int64_t i = bi * 32 + k, a = ba * 32 + tx;
    if (i < In && a < A) tile[k][tx] = src[i * A + a];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {  // write rows a (stride In), i contiguous
    const int64_t a = ba * 32 + k, i = bi * 32 + tx;
    if (i < In && a < A) dst[a * In + i] = tile[tx][k];
  }
}

// ---- cuBLAS through dlopen (the library already depends on torch's CUDA runtime environment; loading by
// SONAME finds the copy torch has loaded)
typedef void* cublas_handle_t;
typedef int (*fn_create)(cublas_handle_t*);
typedef int (*fn_set_stream)(cublas_handle_t, cudaStream_t);
typedef int (*fn_sgemm)(cublas_handle_t, int, int, int, int, int, const float*, const float*, int, const float*, int,
                        const float*, float*, int);
typedef int (*fn_set_math)(cublas_handle_t, int);
struct CublasApi {
  void* h = nullptr;
  fn_create create = nullptr;
  fn_set_stream set_stream = nullptr;
  fn_sgemm sgemm = nullptr;
  fn_set_math set_math = nullptr;
  cublas_handle_t handle[64] = {};
};
enum { kCublasOpN = 0, kCublasOpT = 1, kCublasDefaultMath = 0 };
std::mutex g_cublas_mu;

CublasApi* cublas() {
  static CublasApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libcublas.so.12", "libcublas.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (api.h) {
      api.create = reinterpret_cast<fn_create>(dlsym(api.h, "cublasCreate_v2"));
      api.set_stream = reinterpret_cast<fn_set_stream>(dlsym(api.h, "cublasSetStream_v2"));
      api.sgemm = reinterpret_cast<fn_sgemm>(dlsym(api.h, "cublasSgemm_v2"));
      api.set_math = reinterpret_cast<fn_set_math>(dlsym(api.h, "cublasSetMathMode"));
    }
  });
  if (!api.h || !api.create || !api.set_stream || !api.sgemm) return nullptr;
  return &api;
}

}  // namespace

size_t gaussian_sketch_ws_bytes(const Dims& g, int n) { return n == 0 ? 0 : align_up(g.N * sizeof(float), 256); }

int gaussian_sketch_mode(const float* X, const Dims& g, int n, const float* omega_dense, int R, float* Y, Arena& ar,
                         cudaStream_t s) {
  CublasApi* api = cublas();
  if (!api) {
    set_error("libcublas.so.12 could not be loaded (dense-Gaussian baseline)");
    return KRP_EUNSUPPORTED;
  }
  int dev = 0;
  KRP_CHECK_CUDA(cudaGetDevice(&dev));
  cublas_handle_t h;
  {
    std::lock_guard<std::mutex> lk(g_cublas_mu);
    if (!api->handle[dev % 64]) {
      if (api->create(&api->handle[dev % 64]) != 0) {
        set_error("cublasCreate failed");
        return KRP_ECUDA;
      }
      if (api->set_math) api->set_math(api->handle[dev % 64], kCublasDefaultMath);  // plain fp32 SGEMM
    }
    h = api->handle[dev % 64];
  }
  int64_t A = 1, Cc = 1;
  for (int k = 0; k < n; ++k) A *= g.n[k];
  for (int k = n + 1; k < g.d; ++k) Cc *= g.n[k];
  const int64_t In = g.n[n], K = A * Cc;
  const float* U = X;
  const size_t mark = ar.off;
  if (n > 0) {  // the explicit unfolding (the baseline's unfolding step)
    float* Ub = ar.take<float>(g.N);
    if (ar.overflow()) {
      set_error("workspace too small for the unfolding");
      return KRP_ENOMEM;
    }
    const int64_t nblk = Cc * ((In + 31) / 32) * ((A + 31) / 32);
    unfold_kernel<<<static_cast<unsigned>(nblk), 256, 0, s>>>(X, A, In, Cc, Ub);
    KRP_CHECK_LAUNCH();
    U = Ub;
  }
  if (In > INT32_MAX || K > INT32_MAX) {
    set_error("dense-Gaussian baseline: unfolding too large for a 32-bit GEMM");
    ar.off = mark;
    return KRP_ESHAPE;
  }
  // Y^T (R x I_n, col-major ld R) = Omega^T (R x K: the row-major K x R matrix) * U^T (U: col-major I_n x K)
  const float one = 1.f, zero = 0.f;
  std::lock_guard<std::mutex> lk(g_cublas_mu);
  api->set_stream(h, s);
  const int st = api->sgemm(h, kCublasOpN, kCublasOpT, R, static_cast<int>(In), static_cast<int>(K), &one, omega_dense,
                            R, U, static_cast<int>(In), &zero, Y, R);
  ar.off = mark;
  if (st != 0) {
    set_error("cublasSgemm failed (%d)", st);
    return KRP_ECUDA;
  }
  count_launch();
  return KRP_OK;
}

}  // namespace krp
