// krp_linalg.cu — the dense linear algebra around the sketch (off the headline):
//   * CholeskyQR for the thin QR of each sketch Y_n: fp64 Gram,
//     fp64 Cholesky in one CTA, shifted first pass on breakdown, two refinement
//     passes (sCholeskyQR3 / CholeskyQR2 reading, R15).  diag(R) > 0,
//     so Q equals the sign-fixed Householder Q of the oracle.
//   * TTM  Y = X x_n A for the core G = X x_1 Q_1^T ..., the
//     STHOSVD core update, the truncation updates and reconstruction.
//   * mode-n Gram + Jacobi eigensolver: leading left singular vectors of a core
//     unfolding (truncation l -> r, reading R4; Alg. 2 pattern P:118-120).
//   * squared-difference reduction for ||X - X̂||_F.
// All cross-block sums are fixed-order (deterministic); no atomics.
#include <cmath>

#include "krp_common.cuh"
#include "krp_internal.h"

namespace krp {
namespace {

constexpr int kGramMaxR = 64;

// ------------------------------------------------------------------ Gram of a tall-skinny matrix
template <typename T>
__global__ void __launch_bounds__(256) gram_partial_kernel(const T* __restrict__ Y, int64_t rows, int R,
                                                           int64_t rows_per_block, double* __restrict__ partial) {
  __shared__ double tile[32][kGramMaxR + 1];
  const int64_t r_begin = static_cast<int64_t>(blockIdx.x) * rows_per_block;
  const int64_t r_end = min(rows, r_begin + rows_per_block);
  const int npairs = R * R;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int64_t rb = r_begin; rb < r_end; rb += 32) {
    for (int e = threadIdx.x; e < 32 * R; e += blockDim.x) {
      const int rr = e / R, c = e % R;
      const int64_t row = rb + rr;
      tile[rr][c] = row < r_end ? static_cast<double>(Y[row * R + c]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int pidx = threadIdx.x + q * 256;
      if (pidx < npairs) {
        const int a = pidx / R, b = pidx % R;
        double s = 0.0;
        for (int rr = 0; rr < 32; ++rr) s = fma(tile[rr][a], tile[rr][b], s);
        acc[q] += s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int pidx = threadIdx.x + q * 256;
    if (pidx < npairs) partial[static_cast<int64_t>(blockIdx.x) * npairs + pidx] = acc[q];
  }
}

__global__ void sum_partials_f64_kernel(const double* __restrict__ partial, int P, int64_t len,
                                        double* __restrict__ out) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= len) return;
  double s = 0.0;
  for (int p = 0; p < P; ++p) s += partial[static_cast<int64_t>(p) * len + idx];
  out[idx] = s;
}

// ------------------------------------------------------------------ Cholesky + triangular inverse
// G (R x R, fp64) = L L^T.  Writes Linv (R x R row-major, lower) so that Q = Y Linv^T.
// allow_shift: on breakdown, retry with G + s I, s = 11 (rows R + R(R+1)) u ||Y||_F^2 (flag |= 1);
// a breakdown that cannot be shifted sets flag |= 2.
__global__ void __launch_bounds__(128) chol_inv_kernel(const double* __restrict__ G, int R, int64_t rows,
                                                       double* __restrict__ Linv_out, int* flag, int allow_shift) {
  extern __shared__ double dyn_smem[];
  double(*A)[kGramMaxR + 1] = reinterpret_cast<double(*)[kGramMaxR + 1]>(dyn_smem);
  double(*Li)[kGramMaxR + 1] = reinterpret_cast<double(*)[kGramMaxR + 1]>(dyn_smem + kGramMaxR * (kGramMaxR + 1));
  __shared__ int fail;
  __shared__ double shift;
  const int tid = threadIdx.x;
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < R; ++i) tr += G[i * R + i];
    shift = 0.0;
    (void)tr;
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    __syncthreads();
    for (int e = tid; e < R * R; e += blockDim.x) {
      const int i = e / R, j = e % R;
      A[i][j] = G[e] + (i == j ? shift : 0.0);
    }
    if (tid == 0) fail = 0;
    __syncthreads();
    for (int j = 0; j < R; ++j) {
      if (tid == 0) {
        double dgl = A[j][j];
        for (int k = 0; k < j; ++k) dgl -= A[j][k] * A[j][k];
        if (!(dgl > 0.0) || !isfinite(dgl)) {
          fail = 1;
        } else {
          A[j][j] = sqrt(dgl);
        }
      }
      __syncthreads();
      if (fail) break;
      for (int i = j + 1 + tid; i < R; i += blockDim.x) {
        double v = A[i][j];
        for (int k = 0; k < j; ++k) v -= A[i][k] * A[j][k];
        A[i][j] = v / A[j][j];
      }
      __syncthreads();
    }
    __syncthreads();
    if (!fail) break;
    if (!allow_shift || attempt == 1) {
      if (tid == 0) atomicOr(flag, 2);
      break;
    }
    if (tid == 0) {
      double tr = 0.0;
      for (int i = 0; i < R; ++i) tr += G[i * R + i];
      shift = 11.0 * (static_cast<double>(rows) * R + static_cast<double>(R) * (R + 1)) * 1.1102230246251565e-16 * tr;
      atomicOr(flag, 1);
    }
  }
  __syncthreads();
  if (fail) {
    for (int e = tid; e < R * R; e += blockDim.x) Linv_out[e] = 0.0;
    return;
  }
  // column c of L^{-1} by forward substitution (one thread per column)
  for (int c = tid; c < R; c += blockDim.x) {
    for (int i = 0; i < R; ++i) Li[i][c] = 0.0;
    for (int i = c; i < R; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= A[i][k] * Li[k][c];
      Li[i][c] = s / A[i][i];
    }
  }
  __syncthreads();
  for (int e = tid; e < R * R; e += blockDim.x) Linv_out[e] = Li[e / R][e % R];
}

// Q[i][a] = sum_{b <= a} Y[i][b] * Linv[a][b]
template <typename T>
__global__ void apply_linv_kernel(const T* __restrict__ Y, int64_t rows, int R, const double* __restrict__ Linv,
                                  double* __restrict__ Qd, float* __restrict__ Qf) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * R) return;
  const int64_t i = idx / R;
  const int a = static_cast<int>(idx % R);
  double s = 0.0;
  for (int b = 0; b <= a; ++b) s = fma(static_cast<double>(Y[i * R + b]), Linv[a * R + b], s);
  if (Qd) Qd[idx] = s;
  if (Qf) Qf[idx] = static_cast<float>(s);
}

__global__ void jacobi_top_kernel(const double* __restrict__ Hm, int J, int r, float* __restrict__ U);
constexpr size_t kSquareSmem = 2 * kGramMaxR * (kGramMaxR + 1) * sizeof(double);
int set_square_smem_attrs() {
  static int done = 0;
  if (!done) {
    KRP_CHECK_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kSquareSmem)));
    KRP_CHECK_CUDA(cudaFuncSetAttribute(jacobi_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kSquareSmem)));
    done = 1;
  }
  return KRP_OK;
}

struct GramPlan {
  int P;
  int64_t rows_per_block;
};
GramPlan plan_gram(int64_t rows) {
  GramPlan g;
  int64_t P = (rows + 127) / 128;
  if (P > 256) P = 256;
  if (P < 1) P = 1;
  g.rows_per_block = ((rows + P - 1) / P + 31) / 32 * 32;
  g.P = static_cast<int>((rows + g.rows_per_block - 1) / g.rows_per_block);
  if (g.P < 1) g.P = 1;
  return g;
}

template <typename T>
int gram(const T* Y, int64_t rows, int R, double* G, double* partial, cudaStream_t s) {
  GramPlan gp = plan_gram(rows);
  gram_partial_kernel<T><<<gp.P, 256, 0, s>>>(Y, rows, R, gp.rows_per_block, partial);
  KRP_CHECK_LAUNCH();
  const int64_t len = static_cast<int64_t>(R) * R;
  sum_partials_f64_kernel<<<static_cast<unsigned>((len + 255) / 256), 256, 0, s>>>(partial, gp.P, len, G);
  KRP_CHECK_LAUNCH();
  return KRP_OK;
}

// ------------------------------------------------------------------ TTM
// Y[l + L*(j + J*h)] = sum_i A[j*sj + i*si] * X[l + L*(i + I*h)]  (j in [j0, j0+64))
__global__ void __launch_bounds__(256) ttm_kernel(const float* __restrict__ X, int64_t L, int64_t I, int64_t H,
                                                  const float* __restrict__ A, int J, int64_t sj, int64_t si,
                                                  float* __restrict__ Y, int j0) {
  __shared__ float Xs[16][64 + 4];
  __shared__ float As[16][64 + 4];
  const int64_t P = L * H;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  for (int64_t i0 = 0; i0 < I; i0 += 16) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      int ii, pp;
      if (L == 1) {
        ii = e % 16;
        pp = e / 16;
      } else {
        pp = e % 64;
        ii = e / 64;
      }
      const int64_t p = p0 + pp, i = i0 + ii;
      float v = 0.f;
      if (p < P && i < I) {
        const int64_t l = p % L, h = p / L;
        v = __ldg(X + l + L * (i + I * h));
      }
      Xs[ii][pp] = v;
    }
    for (int e = threadIdx.x; e < 1024; e += 256) {
      const int ii = e % 16, jj = e / 16;
      const int j = j0 + jj;
      const int64_t i = i0 + ii;
      As[ii][jj] = (j < J && i < I) ? __ldg(A + j * sj + i * si) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int ii = 0; ii < 16; ++ii) {
      float xv[4], av[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xv[a] = Xs[ii][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) av[b] = As[ii][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xv[a], av[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t p = p0 + tx + 16 * a;
    if (p >= P) continue;
    const int64_t l = p % L, h = p / L;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = j0 + ty + 16 * b;
      if (j < J) Y[l + L * (j + static_cast<int64_t>(J) * h)] = acc[a][b];
    }
  }
}

// ------------------------------------------------------------------ mode-n Gram
// H[a][b] = sum over fibers f=(l,h) of T[l + L(a + J h)] T[l + L(b + J h)]
__global__ void __launch_bounds__(256) mode_gram_partial_kernel(const float* __restrict__ T, int64_t L, int J,
                                                                int64_t H, int64_t fibers_per_block,
                                                                double* __restrict__ partial) {
  __shared__ float F[32][kGramMaxR + 1];
  const int64_t nf = L * H;
  const int64_t f_begin = static_cast<int64_t>(blockIdx.x) * fibers_per_block;
  const int64_t f_end = min(nf, f_begin + fibers_per_block);
  const int npairs = J * J;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int64_t fb = f_begin; fb < f_end; fb += 32) {
    for (int e = threadIdx.x; e < 32 * J; e += blockDim.x) {
      int ff, a;
      if (L == 1) {
        a = e % J;
        ff = e / J;
      } else {
        ff = e % 32;
        a = e / 32;
      }
      const int64_t f = fb + ff;
      float v = 0.f;
      if (f < f_end) {
        const int64_t l = f % L, h = f / L;
        v = __ldg(T + l + L * (a + static_cast<int64_t>(J) * h));
      }
      F[ff][a] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int pidx = threadIdx.x + q * 256;
      if (pidx < npairs) {
        const int a = pidx / J, b = pidx % J;
        double s = 0.0;
        for (int ff = 0; ff < 32; ++ff) s = fma(static_cast<double>(F[ff][a]), static_cast<double>(F[ff][b]), s);
        acc[q] += s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int pidx = threadIdx.x + q * 256;
    if (pidx < npairs) partial[static_cast<int64_t>(blockIdx.x) * npairs + pidx] = acc[q];
  }
}

struct MGPlan {
  int P;
  int64_t per_block;
};
MGPlan plan_mode_gram(const Dims& g, int n) {
  const int64_t nf = g.N / g.n[n];
  MGPlan p;
  int64_t P = (nf + 1023) / 1024;
  if (P > 592) P = 592;
  if (P < 1) P = 1;
  p.per_block = ((nf + P - 1) / P + 31) / 32 * 32;
  p.P = static_cast<int>((nf + p.per_block - 1) / p.per_block);
  if (p.P < 1) p.P = 1;
  return p;
}

// ------------------------------------------------------------------ symmetric eigensolver (Jacobi)
__global__ void __launch_bounds__(256) jacobi_top_kernel(const double* __restrict__ Hm, int J, int r,
                                                         float* __restrict__ U) {
  extern __shared__ double dyn_smem[];
  double(*A)[kGramMaxR + 1] = reinterpret_cast<double(*)[kGramMaxR + 1]>(dyn_smem);
  double(*V)[kGramMaxR + 1] = reinterpret_cast<double(*)[kGramMaxR + 1]>(dyn_smem + kGramMaxR * (kGramMaxR + 1));
  __shared__ double cs[kGramMaxR / 2], sn[kGramMaxR / 2];
  __shared__ int pp[kGramMaxR / 2], qq[kGramMaxR / 2];
  __shared__ double offn, totn;
  __shared__ int order[kGramMaxR];
  const int tid = threadIdx.x;
  const int m = J + (J & 1);  // even number of players; index J (if odd J) is a dummy
  for (int e = tid; e < J * J; e += blockDim.x) {
    const int i = e / J, j = e % J;
    A[i][j] = Hm[e];
    V[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    {  // off-diagonal and total squared norms: per-thread partial sums, then a fixed-order warp tree
      __shared__ double part_off[8], part_tot[8];
      double off = 0.0, tot = 0.0;
      for (int e = tid; e < 64 * 64; e += blockDim.x) {
        const int i = e >> 6, j = e & 63;
        if (i >= J || j >= J) continue;
        const double v = A[i][j] * A[i][j];
        tot += v;
        if (i != j) off += v;
      }
      for (int o = 16; o > 0; o >>= 1) {
        off += __shfl_xor_sync(0xffffffffu, off, o);
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
      }
      if ((tid & 31) == 0) {
        part_off[tid >> 5] = off;
        part_tot[tid >> 5] = tot;
      }
      __syncthreads();
      if (tid == 0) {
        double so = 0.0, st = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) so += part_off[w], st += part_tot[w];
        offn = so;
        totn = st;
      }
      __syncthreads();
    }
    // converged when the off-diagonal mass is ~(1e-13)^2 of the total: eigenvectors are then accurate
    // far below the fp32 output precision
    if (!(offn > 1e-26 * totn) || m < 2) break;
    for (int round = 0; round < m - 1; ++round) {
      if (tid < m / 2) {
        int a, b;
        if (tid == 0) {
          a = m - 1;
          b = round;
        } else {
          a = (round + tid) % (m - 1);
          b = (round - tid + (m - 1)) % (m - 1);
        }
        const int p = a < b ? a : b, q = a < b ? b : a;
        pp[tid] = p;
        qq[tid] = q;
        double c = 1.0, s = 0.0;
        if (q < J && A[p][q] != 0.0) {
          const double tau = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
        }
        cs[tid] = c;
        sn[tid] = s;
      }
      __syncthreads();
      // rows: A <- J^T A.  (pair k, column) slots as (e >> 6, e & 63): no integer division (J <= 64)
      for (int e = tid; e < (m / 2) * 64; e += blockDim.x) {
        const int k = e >> 6, col = e & 63;
        const int p = pp[k], q = qq[k];
        if (q >= J || col >= J) continue;
        const double c = cs[k], s = sn[k];
        const double ap = A[p][col], aq = A[q][col];
        A[p][col] = c * ap - s * aq;
        A[q][col] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int e = tid; e < (m / 2) * 64; e += blockDim.x) {
        const int k = e >> 6, row = e & 63;
        const int p = pp[k], q = qq[k];
        if (q >= J || row >= J) continue;
        const double c = cs[k], s = sn[k];
        const double ap = A[row][p], aq = A[row][q];
        A[row][p] = c * ap - s * aq;
        A[row][q] = s * ap + c * aq;
        const double vp = V[row][p], vq = V[row][q];
        V[row][p] = c * vp - s * vq;
        V[row][q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    for (int i = 0; i < J; ++i) order[i] = i;
    for (int t = 0; t < r; ++t) {  // selection of the r largest eigenvalues, descending
      int best = t;
      for (int i = t + 1; i < J; ++i)
        if (A[order[i]][order[i]] > A[order[best]][order[best]]) best = i;
      const int tmp = order[t];
      order[t] = order[best];
      order[best] = tmp;
    }
  }
  __syncthreads();
  for (int e = tid; e < J * r; e += blockDim.x) {
    const int i = e / r, t = e % r;
    U[e] = static_cast<float>(V[i][order[t]]);
  }
}

// ------------------------------------------------------------------ squared differences
__global__ void __launch_bounds__(256) sqdiff_partial_kernel(const float* __restrict__ X, const float* __restrict__ Xh,
                                                             int64_t n, int64_t per_block,
                                                             double* __restrict__ partial) {
  __shared__ double s_d[256], s_x[256];
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * per_block;
  const int64_t b1 = min(n, b0 + per_block);
  double sd = 0.0, sx = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const double x = X[i];
    const double dlt = x - static_cast<double>(Xh[i]);
    sd = fma(dlt, dlt, sd);
    sx = fma(x, x, sx);
  }
  s_d[threadIdx.x] = sd;
  s_x[threadIdx.x] = sx;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_d[threadIdx.x] += s_d[threadIdx.x + w];
      s_x[threadIdx.x] += s_x[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = s_d[0];
    partial[2 * blockIdx.x + 1] = s_x[0];
  }
}

__global__ void sqdiff_final_kernel(const double* __restrict__ partial, int P, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int p = 0; p < P; ++p) {
    a += partial[2 * p];
    b += partial[2 * p + 1];
  }
  out[0] += a;
  out[1] += b;
}

__global__ void copy_cols_kernel(const float* __restrict__ src, int64_t rows, int scols, float* __restrict__ dst,
                                 int dcols) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * dcols) return;
  const int64_t i = idx / dcols;
  const int j = static_cast<int>(idx % dcols);
  dst[idx] = src[i * scols + j];
}

}  // namespace

// ------------------------------------------------------------------ host wrappers
size_t cholqr_ws_bytes(int64_t rows, int R) {
  GramPlan gp = plan_gram(rows);
  size_t b = 0;
  b += 2 * align_up(static_cast<size_t>(rows) * R * sizeof(double), 256);         // two fp64 Q buffers
  b += 2 * align_up(static_cast<size_t>(R) * R * sizeof(double), 256);            // G, Linv
  b += align_up(static_cast<size_t>(gp.P) * R * R * sizeof(double), 256);         // Gram partials
  return b;
}

int cholqr(const float* Y, int64_t rows, int R, float* Qf, double* Qd, int* flag_dev, Arena& ar, cudaStream_t s) {
  if (R > kGramMaxR) {
    set_error("CholeskyQR supports R <= %d (got %d)", kGramMaxR, R);
    return KRP_EINVAL;
  }
  KRP_TRY(set_square_smem_attrs());
  const size_t mark = ar.off;
  GramPlan gp = plan_gram(rows);
  double* Q1 = ar.take<double>(static_cast<size_t>(rows) * R);
  double* Q2 = ar.take<double>(static_cast<size_t>(rows) * R);
  double* G = ar.take<double>(static_cast<size_t>(R) * R);
  double* Li = ar.take<double>(static_cast<size_t>(R) * R);
  double* part = ar.take<double>(static_cast<size_t>(gp.P) * R * R);
  if (ar.overflow()) {
    set_error("workspace too small for CholeskyQR");
    return KRP_ENOMEM;
  }
  const int64_t tot = rows * R;
  const unsigned nb = static_cast<unsigned>((tot + 255) / 256);
  // pass 1 (shift allowed)
  KRP_TRY(gram<float>(Y, rows, R, G, part, s));
  chol_inv_kernel<<<1, 128, kSquareSmem, s>>>(G, R, rows, Li, flag_dev, 1);
  KRP_CHECK_LAUNCH();
  apply_linv_kernel<float><<<nb, 256, 0, s>>>(Y, rows, R, Li, Q1, nullptr);
  KRP_CHECK_LAUNCH();
  // pass 2
  KRP_TRY(gram<double>(Q1, rows, R, G, part, s));
  chol_inv_kernel<<<1, 128, kSquareSmem, s>>>(G, R, rows, Li, flag_dev, 0);
  KRP_CHECK_LAUNCH();
  apply_linv_kernel<double><<<nb, 256, 0, s>>>(Q1, rows, R, Li, Q2, nullptr);
  KRP_CHECK_LAUNCH();
  // pass 3 (restores orthogonality after a shifted first pass; a no-op refinement otherwise)
  KRP_TRY(gram<double>(Q2, rows, R, G, part, s));
  chol_inv_kernel<<<1, 128, kSquareSmem, s>>>(G, R, rows, Li, flag_dev, 0);
  KRP_CHECK_LAUNCH();
  apply_linv_kernel<double><<<nb, 256, 0, s>>>(Q2, rows, R, Li, Qd, Qf);
  KRP_CHECK_LAUNCH();
  ar.off = mark;
  return KRP_OK;
}

int ttm(const float* X, const Dims& g, int n, const float* A, int J, int64_t sj, int64_t si, float* Y,
        cudaStream_t s) {
  const int64_t L = g.stride[n], I = g.n[n], H = g.N / (L * I);
  const int64_t P = L * H;
  const unsigned nb = static_cast<unsigned>((P + 63) / 64);
  for (int j0 = 0; j0 < J; j0 += 64) {
    ttm_kernel<<<nb, 256, 0, s>>>(X, L, I, H, A, J, sj, si, Y, j0);
    KRP_CHECK_LAUNCH();
  }
  return KRP_OK;
}

size_t mode_gram_ws_bytes(const Dims& g, int n) {
  MGPlan p = plan_mode_gram(g, n);
  return align_up(static_cast<size_t>(p.P) * g.n[n] * g.n[n] * sizeof(double), 256);
}

int mode_gram(const float* T, const Dims& g, int n, double* H, Arena& ar, cudaStream_t s) {
  const int J = static_cast<int>(g.n[n]);
  if (J > kGramMaxR) {
    set_error("mode Gram supports size <= %d (got %d)", kGramMaxR, J);
    return KRP_EINVAL;
  }
  MGPlan p = plan_mode_gram(g, n);
  const size_t mark = ar.off;
  double* part = ar.take<double>(static_cast<size_t>(p.P) * J * J);
  if (ar.overflow()) {
    set_error("workspace too small for mode Gram");
    return KRP_ENOMEM;
  }
  const int64_t L = g.stride[n], Hh = g.N / (L * J);
  mode_gram_partial_kernel<<<p.P, 256, 0, s>>>(T, L, J, Hh, p.per_block, part);
  KRP_CHECK_LAUNCH();
  const int64_t len = static_cast<int64_t>(J) * J;
  sum_partials_f64_kernel<<<static_cast<unsigned>((len + 255) / 256), 256, 0, s>>>(part, p.P, len, H);
  KRP_CHECK_LAUNCH();
  ar.off = mark;
  return KRP_OK;
}

int sym_eig_top(const double* H, int J, int r, float* U, cudaStream_t s) {
  if (J > kGramMaxR || r > J) {
    set_error("eigensolver: J=%d r=%d unsupported", J, r);
    return KRP_EINVAL;
  }
  KRP_TRY(set_square_smem_attrs());
  jacobi_top_kernel<<<1, 256, kSquareSmem, s>>>(H, J, r, U);
  KRP_CHECK_LAUNCH();
  return KRP_OK;
}

size_t sqdiff_ws_bytes(int64_t n) { return align_up(2 * 1184 * sizeof(double), 256); }

int sqdiff_accumulate(const float* X, const float* Xh, int64_t n, double* out, Arena& ar, cudaStream_t s) {
  int64_t P = (n + 65535) / 65536;
  if (P > 1184) P = 1184;
  if (P < 1) P = 1;
  const int64_t per = (n + P - 1) / P;
  P = (n + per - 1) / per;
  if (P < 1) P = 1;
  const size_t mark = ar.off;
  double* part = ar.take<double>(2 * 1184);
  if (ar.overflow()) {
    set_error("workspace too small for the error pass");
    return KRP_ENOMEM;
  }
  sqdiff_partial_kernel<<<static_cast<unsigned>(P), 256, 0, s>>>(X, Xh, n, per, part);
  KRP_CHECK_LAUNCH();
  sqdiff_final_kernel<<<1, 32, 0, s>>>(part, static_cast<int>(P), out);
  KRP_CHECK_LAUNCH();
  ar.off = mark;
  return KRP_OK;
}

int copy_cols(const float* src, int64_t rows, int scols, float* dst, int dcols, cudaStream_t s) {
  const int64_t tot = rows * dcols;
  copy_cols_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(src, rows, scols, dst, dcols);
  KRP_CHECK_LAUNCH();
  return KRP_OK;
}

}  // namespace krp
