// krp_internal.h — internal entry points between the translation units of libkrp.
#pragma once
#include "krp_common.cuh"

namespace krp {

// ---- the sketch (krp_sketch_tc.cu): tcgen05 3xTF32 kernels for every shape; want_mode[k] selects which
// Y_k are produced.  R in [1, 256] (column groups of <= 64 per launch).  KRP_EUNSUPPORTED (nothing
// launched) on a device that is not sm_100a.
bool tc_device_ok();
void* tma_encode_fn();  // the driver's cuTensorMapEncodeTiled (PFN_cuTensorMapEncodeTiled_v12000)
int device_sms();       // SM count of the current device
size_t tc_sketch_ws_bytes(const Dims& g, int R, const bool* want_mode);
int tc_sketch(const float* X, const Dims& g, const OmegaPtrs& om, int R, const bool* want_mode, float* const* Y,
              Arena& ar, cudaStream_t s);
inline size_t sketch_ws_bytes(const Dims& g, int R, const bool* want_mode) { return tc_sketch_ws_bytes(g, R, want_mode); }
inline int sketch(const float* X, const Dims& g, const OmegaPtrs& om, int R, const bool* want_mode, float* const* Y,
                  Arena& ar, cudaStream_t s) {
  return tc_sketch(X, g, om, R, want_mode, Y, ar, s);
}

// ---- the paper's dense-Gaussian baseline sketch (krp_baselines.cu): Y = X_(n) Omega_dense, Omega_dense
// (N/I_n) x R row-major in the column order of X_(n); explicit unfolding + fp32 SGEMM (cuBLAS via dlopen)
size_t gaussian_sketch_ws_bytes(const Dims& g, int n);
int gaussian_sketch_mode(const float* X, const Dims& g, int n, const float* omega_dense, int R, float* Y, Arena& ar,
                         cudaStream_t s);

// ---- NEXT-4: randomized HOSVD of the Hadamard product of two 3-way Tucker tensors (krp_hadamard.cu, Alg. 9)
int hadamard_tucker_impl(const float* F, const int64_t* q, const float* const* A, const float* G, const int64_t* s,
                         const float* const* U, const int64_t* n, const int* ranks, const int* ls,
                         const float* const* omega, float* const* Qout, float* core, Arena& ar, cudaStream_t st,
                         bool measure_only);

// ---- dense linear algebra (krp_linalg.cu)
// CholeskyQR with shifted first pass and two refinement passes (sCholeskyQR3; plain CholeskyQR2
// when the first Cholesky succeeds without shift).  Y: rows x R fp32 row-major.
// Writes Q (rows x R) as fp32 (Qf, may be null) and fp64 (Qd, may be null).
size_t cholqr_ws_bytes(int64_t rows, int R);
int cholqr(const float* Y, int64_t rows, int R, float* Qf, double* Qd, int* flag_dev, Arena& ar, cudaStream_t s);

// Y = X x_n A for X of dims g (fp32), A: J x I_n with element (j, i) at A[j*sj + i*si] (fp32).
// With an arena holding ttm_ws_bytes(g, n, J), mode 0 runs on the tensor cores (ttm0_tc, 3xTF32);
// otherwise (and for every other mode) on the fp32 FMA kernels.
size_t ttm_ws_bytes(const Dims& g, int n, int J);
int ttm(const float* X, const Dims& g, int n, const float* A, int J, int64_t sj, int64_t si, float* Y,
        cudaStream_t s, Arena* ar = nullptr);

// ---- mode-0 TTM on tcgen05 (krp_ttm_tc.cu): Y[j + J h] = sum_i A[j sj + i si] X[i + I h], J <= 64,
// I % 4 == 0, X 16-byte aligned; workspace: the B-operand image of A.  H1 > 0 (dividing H): the output is
// written mode-permuted, Y[h1 + H1 (j + J h2)] for h = h1 + H1 h2, i.e. (I_2, J, I_3..) instead of
// (J, I_2, I_3..), so the next contraction (over I_2) is again a mode-0 product.
// gram_partials (J <= 32, unpermuted): also writes 4 per-CTA partials of the output's mode-1 Gram
// Y_(1) Y_(1)ᵀ (fp64, J x J each, ttm0_tc_grid(H) * 4 of them) for a fixed-order sum.
bool ttm0_tc_ok(const float* X, int64_t I, int64_t H, int J);
size_t ttm0_tc_ws_bytes(int64_t I, int J);
int ttm0_tc_grid(int64_t H);
int ttm0_tc(const float* X, int64_t I, int64_t H, const float* A, int J, int64_t sj, int64_t si, float* Y, Arena& ar,
            cudaStream_t s, int64_t H1 = 0, double* gram_partials = nullptr);
// out[idx] = sum_p partial[p * len + idx], fixed order (krp_linalg.cu)
int sum_partials_f64(const double* partial, int P, int64_t len, double* out, cudaStream_t s);

// H = T_(n) T_(n)^T (J x J, fp64) for T of dims g with J = g.n[n].
size_t mode_gram_ws_bytes(const Dims& g, int n);
int mode_gram(const float* T, const Dims& g, int n, double* H, Arena& ar, cudaStream_t s);

// Leading r eigenvectors (descending eigenvalues) of a symmetric J x J fp64 matrix (J <= 64),
// written as U (J x r row-major) in fp32.
int sym_eig_top(const double* H, int J, int r, float* U, cudaStream_t s);
// count independent problems in one launch (one block each): H[k] (J x J) -> U[k] (J x r[k])
int sym_eig_top_batched(const double* const* H, int count, int J, const int* r, float* const* U, cudaStream_t s);

// sum (X - Xh)^2 and sum X^2 over n elements, fp64, fixed order; out[0], out[1] accumulate (+=).
size_t sqdiff_ws_bytes(int64_t n);
int sqdiff_accumulate(const float* X, const float* Xh, int64_t n, double* out, Arena& ar, cudaStream_t s);

// row-major matrix copy with column subset: dst[i*dcols + j] = src[i*scols + j], j < dcols
int copy_cols(const float* src, int64_t rows, int scols, float* dst, int dcols, cudaStream_t s);

}  // namespace krp
