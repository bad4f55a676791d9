// krp_hadamard.cu — NEXT-4: randomized HOSVD of the Hadamard product of two 3-way Tucker tensors (App. C,
// Alg. 9; Kressner & Perisa's recompression, analysed by Theorem 5.1).
//
// Z = X ∗ Y with X = F ×_n A_n, Y = G ×_n U_n is never formed.  With H = F ⊗ G (q_n s_n per mode) and
// the row-wise Kronecker factors A_n ⊙ᵀ U_n, Z = H ×_n (A_n ⊙ᵀ U_n) (eq. C.1), so for each mode i:
//   M_j  = (A_jᵀ ⊙ U_jᵀ) Ω_{i,j}              (q_j s_j x l_i; kr_project_kernel, n_j-length dots)
//   T_i  = H_(i) (M_k ⊙ M_j)                  (q_i s_i x l_i: the KRP sketch of the small tensor H — the
//                                              tcgen05 sketch kernel, one mode, this mode's own factors)
//   Ẑ_i  = (A_i ⊙ᵀ U_i) T_i                   (n_i x l_i; row_kron_apply_kernel)
//   Q_i  = CholeskyQR2(Ẑ_i)
// then H ×_n P_n with P_n = Q_nᵀ (A_n ⊙ᵀ U_n) (kr_project_kernel again, with Q_n for Ω) through the TTM
// kernels, and for r_n < l_n the HOSVD truncation of that core (reading R4 applied to Alg. 9).
#include <algorithm>

#include "krp_common.cuh"
#include "krp_internal.h"

namespace krp {
namespace {

// H(A, B, C) = F(a,b,c) G(alpha,beta,gamma), A = alpha + a * s1 (P:960-962, 0-based), first index fastest.
__global__ void tensor_kron_kernel(const float* __restrict__ F, int64_t q1, int64_t q2, int64_t q3,
                                   const float* __restrict__ G, int64_t s1, int64_t s2, int64_t s3,
                                   float* __restrict__ H) {
  const int64_t n1 = q1 * s1, n2 = q2 * s2, n3 = q3 * s3, tot = n1 * n2 * n3;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < tot;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i1 = e % n1, r = e / n1, i2 = r % n2, i3 = r / n2;
    const int64_t a = i1 / s1, al = i1 % s1, b = i2 / s2, be = i2 % s2, c = i3 / s3, ga = i3 % s3;
    H[e] = F[a + q1 * (b + q2 * c)] * G[al + s1 * (be + s2 * ga)];
  }
}

// M((a,alpha), r) = Σ_k A(k,a) U(k,alpha) Om(k,r)   [(Aᵀ ⊙ Uᵀ) Om], rows a*s + alpha; fp64 sums.
// A: n x q, U: n x s row-major; Om: n x l with row stride ldo; M: (q s) x l row-major.
__global__ void kr_project_kernel(const float* __restrict__ A, int q, const float* __restrict__ U, int s, int64_t n,
                                  const float* __restrict__ Om, int ldo, int l, float* __restrict__ M) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(q) * s * l) return;
  const int r = static_cast<int>(e % l);
  const int64_t row = e / l;
  const int a = static_cast<int>(row / s), al = static_cast<int>(row % s);
  double acc = 0.0;
  for (int64_t k = 0; k < n; ++k)
    acc += static_cast<double>(A[k * q + a]) * U[k * s + al] * Om[k * ldo + r];
  M[e] = static_cast<float>(acc);
}

// Ẑ(i, r) = Σ_{a,alpha} A(i,a) U(i,alpha) T((a,alpha), r)   [(A ⊙ᵀ U) T]; fp64 sums.
__global__ void row_kron_apply_kernel(const float* __restrict__ A, int q, const float* __restrict__ U, int s,
                                      int64_t n, const float* __restrict__ T, int l, float* __restrict__ Z) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * l) return;
  const int r = static_cast<int>(e % l);
  const int64_t i = e / l;
  double acc = 0.0;
  for (int a = 0; a < q; ++a) {
    const double av = A[i * q + a];
    double inner = 0.0;
    for (int al = 0; al < s; ++al) inner += static_cast<double>(U[i * s + al]) * T[(static_cast<int64_t>(a) * s + al) * l + r];
    acc += av * inner;
  }
  Z[e] = static_cast<float>(acc);
}

unsigned blocks_for(int64_t n, int t = 256) { return static_cast<unsigned>(std::min<int64_t>((n + t - 1) / t, 1 << 20)); }

}  // namespace

// Workspace and launch sequence (d = 3).  measure_only: only the arena is sized.
int hadamard_tucker_impl(const float* F, const int64_t* q, const float* const* A, const float* G, const int64_t* s,
                         const float* const* U, const int64_t* n, const int* ranks, const int* ls,
                         const float* const* omega, float* const* Qout, float* core, Arena& ar, cudaStream_t st,
                         bool measure_only) {
  constexpr int d = 3;
  int64_t hd[d];
  int lmax = 0;
  for (int k = 0; k < d; ++k) {
    hd[k] = q[k] * s[k];
    lmax = std::max(lmax, ls[k]);
  }
  const Dims hg = make_dims(d, hd);
  float* H = ar.take<float>(hg.N);
  float* M[d];
  for (int k = 0; k < d; ++k) M[k] = ar.take<float>(hd[k] * lmax);
  float* T = ar.take<float>(*std::max_element(hd, hd + d) * lmax);
  float* Zh[d];
  float* Qf[d];
  for (int k = 0; k < d; ++k) {
    Zh[k] = ar.take<float>(n[k] * ls[k]);
    Qf[k] = ar.take<float>(n[k] * ls[k]);
  }
  float* P[d];
  for (int k = 0; k < d; ++k) P[k] = ar.take<float>(hd[k] * ls[k]);
  int* flag = ar.take<int>(d);
  // TTM chain buffers: H -> (l1, n2h, n3h) -> (l1, l2, n3h) -> core (l1, l2, l3)
  const int64_t c1 = ls[0] * hd[1] * hd[2], c2 = static_cast<int64_t>(ls[0]) * ls[1] * hd[2];
  const int64_t lcore = static_cast<int64_t>(ls[0]) * ls[1] * ls[2];
  float* B1 = ar.take<float>(std::max(c1, lcore));
  float* B2 = ar.take<float>(std::max(c2, lcore));
  double* Hg = ar.take<double>(static_cast<size_t>(d) * lmax * lmax);
  float* Ue = ar.take<float>(static_cast<size_t>(d) * lmax * lmax);
  size_t scratch = 0;
  for (int i = 0; i < d; ++i) {
    bool want[kMaxD] = {};
    want[i] = true;
    scratch = std::max(scratch, sketch_ws_bytes(hg, ls[i], want));
    scratch = std::max(scratch, cholqr_ws_bytes(n[i], ls[i]));
  }
  {
    int64_t cd[d] = {ls[0], ls[1], ls[2]};
    for (int i = 0; i < d; ++i) scratch = std::max(scratch, mode_gram_ws_bytes(make_dims(d, cd), i));
  }
  const size_t mark = ar.off;
  ar.take<char>(scratch);
  if (measure_only) return KRP_OK;
  if (ar.overflow()) {
    set_error("workspace too small for krp_hadamard_tucker");
    return KRP_ENOMEM;
  }
  ar.off = mark;
  KRP_CHECK_CUDA(cudaMemsetAsync(flag, 0, d * sizeof(int), st));
  // H = F ⊗ G (the small Kronecker core; Z itself is never formed)
  tensor_kron_kernel<<<blocks_for(hg.N), 256, 0, st>>>(F, q[0], q[1], q[2], G, s[0], s[1], s[2], H);
  KRP_CHECK_LAUNCH();
  for (int i = 0; i < d; ++i) {
    const int l = ls[i];
    // M_j = (A_jᵀ ⊙ U_jᵀ) Ω_{i,j} for the other two modes
    OmegaPtrs om{};
    for (int j = 0; j < d; ++j) {
      if (j == i) continue;
      kr_project_kernel<<<blocks_for(hd[j] * l), 256, 0, st>>>(A[j], static_cast<int>(q[j]), U[j], static_cast<int>(s[j]),
                                                               n[j], omega[i * d + j], l, l, M[j]);
      KRP_CHECK_LAUNCH();
      om.p[j] = M[j];
    }
    // T_i = H_(i) (M_k ⊙ M_j): the KRP sketch of H in mode i with this mode's factors
    bool want[kMaxD] = {};
    want[i] = true;
    float* Yp[kMaxD] = {};
    Yp[i] = T;
    KRP_TRY(sketch(H, hg, om, l, want, Yp, ar, st));
    ar.off = mark;
    // Ẑ_i = (A_i ⊙ᵀ U_i) T_i, then Q_i = orth(Ẑ_i)
    row_kron_apply_kernel<<<blocks_for(n[i] * l), 256, 0, st>>>(A[i], static_cast<int>(q[i]), U[i], static_cast<int>(s[i]),
                                                                n[i], T, l, Zh[i]);
    KRP_CHECK_LAUNCH();
    KRP_TRY(cholqr(Zh[i], n[i], l, Qf[i], nullptr, flag + i, ar, st));
    ar.off = mark;
    // P_iᵀ = (A_iᵀ ⊙ U_iᵀ) Q_i  (q_i s_i x l)
    kr_project_kernel<<<blocks_for(hd[i] * l), 256, 0, st>>>(A[i], static_cast<int>(q[i]), U[i], static_cast<int>(s[i]),
                                                             n[i], Qf[i], l, l, P[i]);
    KRP_CHECK_LAUNCH();
  }
  // core (l1, l2, l3) = H ×_1 P_1 ×_2 P_2 ×_3 P_3  (A = P_i: (j, k) at P_iᵀ[k * l + j])
  KRP_TRY(ttm(H, hg, 0, P[0], ls[0], 1, ls[0], B1, st));
  int64_t d1[d] = {ls[0], hd[1], hd[2]};
  KRP_TRY(ttm(B1, make_dims(d, d1), 1, P[1], ls[1], 1, ls[1], B2, st));
  int64_t d2[d] = {ls[0], ls[1], hd[2]};
  KRP_TRY(ttm(B2, make_dims(d, d2), 2, P[2], ls[2], 1, ls[2], B1, st));
  // truncation l -> r by the HOSVD of the core (R4)
  int64_t cd[d] = {ls[0], ls[1], ls[2]};
  const Dims c0 = make_dims(d, cd);
  const double* Hk[kMaxD];
  float* Uk[kMaxD];
  int rk[kMaxD];
  int neig = 0;
  bool trunc[d] = {false, false, false};
  for (int i = 0; i < d; ++i) {
    if (ranks[i] < ls[i]) {
      if (ls[i] != lmax) {  // the batched eigensolver takes one matrix size
        set_error("krp_hadamard_tucker: truncation needs equal sketch widths l_i");
        return KRP_EINVAL;
      }
      KRP_TRY(mode_gram(B1, c0, i, Hg + static_cast<size_t>(i) * lmax * lmax, ar, st));
      ar.off = mark;
      Hk[neig] = Hg + static_cast<size_t>(i) * lmax * lmax;
      Uk[neig] = Ue + static_cast<size_t>(i) * lmax * lmax;
      rk[neig] = ranks[i];
      ++neig;
      trunc[i] = true;
    }
  }
  if (neig > 0) KRP_TRY(sym_eig_top_batched(Hk, neig, lmax, rk, Uk, st));
  float* Gc = B1;
  float* Gn = B2;
  for (int i = 0; i < d; ++i) {
    if (trunc[i]) {
      const float* Um = Ue + static_cast<size_t>(i) * lmax * lmax;
      int64_t qd[2] = {ls[i], n[i]};
      KRP_TRY(ttm(Qf[i], make_dims(2, qd), 0, Um, ranks[i], 1, ranks[i], Qout[i], st));
      KRP_TRY(ttm(Gc, make_dims(d, cd), i, Um, ranks[i], 1, ranks[i], Gn, st));
      std::swap(Gc, Gn);
      cd[i] = ranks[i];
    } else {
      KRP_CHECK_CUDA(cudaMemcpyAsync(Qout[i], Qf[i], n[i] * ls[i] * sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
  }
  KRP_CHECK_CUDA(cudaMemcpyAsync(core, Gc, static_cast<size_t>(cd[0]) * cd[1] * cd[2] * sizeof(float),
                                 cudaMemcpyDeviceToDevice, st));
  int hflag[d] = {};
  KRP_CHECK_CUDA(cudaMemcpyAsync(hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, st));
  KRP_CHECK_CUDA(cudaStreamSynchronize(st));
  if ((hflag[0] | hflag[1] | hflag[2]) & 2) {
    set_error("CholeskyQR breakdown (shifted fallback failed)");
    return KRP_ENUMERIC;
  }
  return KRP_OK;
}

}  // namespace krp
