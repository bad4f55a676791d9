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
#include <cstdlib>

#include "krp_common.cuh"
#include "krp_internal.h"

namespace krp {
namespace {

constexpr int kGramMaxR = 64;

// ------------------------------------------------------------------ Gram of a tall-skinny matrix
template <typename T>
__global__ void __launch_bounds__(256) gram_partial_kernel(const T* __restrict__ Y, int64_t rows, int R,
                                                           int64_t rows_per_block, double* __restrict__ partial,
                                                           const int* __restrict__ gate = nullptr) {
  if (gate && !(*gate & 1)) return;
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

// gate (optional): run only if *gate & 1 (the shifted first CholeskyQR pass happened)
// out[idx] = sum_p partial[p * len + idx] in a fixed order: warp w of the block sums p = w, w+32, ... for
// 32 consecutive idx (coalesced; four independent chains so four loads are in flight), and warp 0 adds the
// 32 warp sums in order w = 0..31.  Launch: ceil(len/32) blocks of 1024 threads.
__global__ void __launch_bounds__(1024) sum_partials_f64_kernel(const double* __restrict__ partial, int P,
                                                                int64_t len, double* __restrict__ out,
                                                                const int* __restrict__ gate = nullptr) {
  __shared__ double ws[32][33];
  if (gate && !(*gate & 1)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (idx < len) {
    const double* src = partial + idx;
    int p = w;
    for (; p + 96 < P; p += 128) {
      s0 += src[static_cast<int64_t>(p) * len];
      s1 += src[static_cast<int64_t>(p + 32) * len];
      s2 += src[static_cast<int64_t>(p + 64) * len];
      s3 += src[static_cast<int64_t>(p + 96) * len];
    }
    for (; p < P; p += 32) s0 += src[static_cast<int64_t>(p) * len];
  }
  ws[w][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (w == 0 && idx < len) {
    double t = 0.0;
    for (int k = 0; k < 32; ++k) t += ws[k][lane];
    out[idx] = t;
  }
}

// ------------------------------------------------------------------ Cholesky + triangular inverse
// G (R x R, fp64) = L L^T.  Writes Linv (R x R row-major, lower) so that Q = Y Linv^T.
// allow_shift: on breakdown, retry with G + s I, s = 11 (rows R + R(R+1)) u ||Y||_F^2 (flag |= 1);
// a breakdown that cannot be shifted sets flag |= 2.
// allow_shift == 2: the third (refinement) pass — factorise only if the first pass was shifted
// (flag & 1), else write Linv = I so that the pass is an exact copy (plain CholeskyQR2).
__device__ __forceinline__ double rcp_nr_f64(double x) {  // 1 / x: hardware approximation + 2 Newton steps
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  return r * fma(-x, r, 2.0);
}

// Register-resident right-looking Cholesky and triangular inverse, 1024 threads, ONE barrier per step:
// thread t owns the lower-triangle entries e = t, t + 1024, t + 2048 (e = i(i+1)/2 + k, k <= i) in
// registers.  Cholesky step j: column j (unscaled) is final, broadcast through a double-buffered shared
// column (its owners wrote it while finishing step j-1); each owner of (i, k), k > j, subtracts
// a_ij a_kj / a_jj and, if k == j+1, publishes the result for step j+1.  Column scalings L_ij = a_ij /
// sqrt(a_jj) are applied once at the end.  Inverse: rows of U = unscaled L^-1 likewise (step i broadcasts
// row i; U_rc -= (L_ri / L_ii) U_ic), scaled by 1 / L_ii at the end.
constexpr int kCholThreads = 1024, kCholSlots = 3;  // 3 x 1024 >= 64 * 65 / 2
__global__ void __launch_bounds__(kCholThreads) chol_inv_kernel(const double* __restrict__ G, int R, int64_t rows,
                                                                double* __restrict__ Linv_out, int* flag,
                                                                int allow_shift) {
  if (allow_shift == 2 && !(*flag & 1)) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) Linv_out[e] = (e / R == e % R) ? 1.0 : 0.0;
    return;
  }
  if (allow_shift == 2) allow_shift = 0;
  __shared__ double colb[2][kGramMaxR];   // Cholesky: broadcast column; inverse: broadcast row
  __shared__ double Ls[kGramMaxR][kGramMaxR + 1];
  __shared__ double rdiag[kGramMaxR];     // 1 / L_jj
  __shared__ double shift;
  const int tid = threadIdx.x;
  const int ne = R * (R + 1) / 2;
  int ei[kCholSlots], ek[kCholSlots];
#pragma unroll
  for (int u = 0; u < kCholSlots; ++u) {
    const int e = tid + u * kCholThreads;
    int i = static_cast<int>((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) / 2 > e) --i;
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    ei[u] = e < ne ? i : -1;
    ek[u] = e < ne ? e - i * (i + 1) / 2 : -1;
  }
  if (tid == 0) shift = 0.0;
  bool failed = false;
  double a[kCholSlots];
  for (int attempt = 0; attempt < 2; ++attempt) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kCholSlots; ++u) {
      a[u] = ei[u] >= 0 ? G[ei[u] * R + ek[u]] + (ei[u] == ek[u] ? shift : 0.0) : 0.0;
      if (ek[u] == 0) colb[0][ei[u]] = a[u];
    }
    __syncthreads();
    failed = false;
    for (int j = 0; j < R; ++j) {
      const double* col = colb[j & 1];
      double* nxt = colb[(j + 1) & 1];
      const double dgl = col[j];
      if (!(dgl > 0.0) || !isfinite(dgl)) {  // every thread reads the same pivot: a uniform exit
        failed = true;
        break;
      }
      const double rinv = rcp_nr_f64(dgl);
      if (tid == 0) rdiag[j] = rsqrt(dgl);
#pragma unroll
      for (int u = 0; u < kCholSlots; ++u) {
        const int i = ei[u], k = ek[u];
        if (k > j) {
          a[u] = fma(-col[i] * rinv, col[k], a[u]);
          if (k == j + 1) nxt[i] = a[u];
        }
      }
      __syncthreads();
    }
    if (!failed) break;
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
  if (failed) {
    for (int e = tid; e < R * R; e += blockDim.x) Linv_out[e] = 0.0;
    return;
  }
  // L = scaled columns, into shared memory for the inverse
#pragma unroll
  for (int u = 0; u < kCholSlots; ++u)
    if (ei[u] >= 0) Ls[ei[u]][ek[u]] = a[u] * rdiag[ek[u]];
  // U = identity (unscaled inverse), row 0 published
#pragma unroll
  for (int u = 0; u < kCholSlots; ++u) {
    a[u] = (ei[u] >= 0 && ei[u] == ek[u]) ? 1.0 : 0.0;
    if (ei[u] == 0) colb[0][ek[u]] = a[u];
  }
  __syncthreads();
  for (int i = 0; i < R; ++i) {
    const double* row = colb[i & 1];
    double* nxt = colb[(i + 1) & 1];
    const double rd = rdiag[i];
#pragma unroll
    for (int u = 0; u < kCholSlots; ++u) {
      const int r = ei[u], c = ek[u];
      if (r > i && c <= i) a[u] = fma(-Ls[r][i] * rd, row[c], a[u]);
      if (r == i + 1) nxt[c] = a[u];
    }
    __syncthreads();
  }
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int i = e / R, c = e % R;
    if (c > i) Linv_out[e] = 0.0;
  }
#pragma unroll
  for (int u = 0; u < kCholSlots; ++u)
    if (ei[u] >= 0) Linv_out[ei[u] * R + ek[u]] = a[u] * rdiag[ei[u]];
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

struct EigBatch;
__global__ void jacobi_top_kernel(EigBatch batch, int J);
constexpr size_t kSquareSmem = 2 * kGramMaxR * (kGramMaxR + 1) * sizeof(double);
constexpr size_t kJacobiSmem = 3 * kGramMaxR * (kGramMaxR + 1) * sizeof(double);
// The raised shared-memory limits are a per-device function attribute: set on every call (cheap host call),
// so a second device in the process and concurrent host threads see them too.
int set_square_smem_attrs() {
  KRP_CHECK_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kSquareSmem)));
  KRP_CHECK_CUDA(cudaFuncSetAttribute(jacobi_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kJacobiSmem)));
  return KRP_OK;
}

struct GramPlan {
  int P;
  int64_t rows_per_block;
};
GramPlan plan_gram(int64_t rows) {
  GramPlan g;
  int64_t P = (rows + 31) / 32;  // one 32-row tile per block while that fills up to 256 blocks
  if (P > 256) P = 256;
  if (P < 1) P = 1;
  g.rows_per_block = ((rows + P - 1) / P + 31) / 32 * 32;
  g.P = static_cast<int>((rows + g.rows_per_block - 1) / g.rows_per_block);
  if (g.P < 1) g.P = 1;
  return g;
}

template <typename T>
int gram(const T* Y, int64_t rows, int R, double* G, double* partial, cudaStream_t s, const int* gate = nullptr) {
  GramPlan gp = plan_gram(rows);
  gram_partial_kernel<T><<<gp.P, 256, 0, s>>>(Y, rows, R, gp.rows_per_block, partial, gate);
  KRP_CHECK_LAUNCH();
  const int64_t len = static_cast<int64_t>(R) * R;
  sum_partials_f64_kernel<<<static_cast<unsigned>((len + 31) / 32), 1024, 0, s>>>(partial, gp.P, len, G, gate);
  KRP_CHECK_LAUNCH();
  return KRP_OK;
}

// ------------------------------------------------------------------ TTM
// Y[l + L*(j + J*h)] = sum_i A[j*sj + i*si] * X[l + L*(i + I*h)]  (j in [j0, j0+64))
// Generic layout: 64 (l,h) columns x 64 j per block, i in steps of 16.  Each thread's global offsets are
// fixed across the i loop, so the (l, h) decomposition is done once; the next i step is prefetched into
// registers while the current one is multiplied.
template <int JB>  // j per thread (j tile = 16 JB)
__global__ void __launch_bounds__(256) ttm_kernel(const float* __restrict__ X, int64_t L, int64_t I, int64_t H,
                                                  const float* __restrict__ A, int J, int64_t sj, int64_t si,
                                                  float* __restrict__ Y, int j0) {
  __shared__ float Xs[16][64 + 4];
  __shared__ float As[16][16 * JB + 4];
  const int64_t P = L * H;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  int xi[4], xp[4], ai[JB], aj[JB];
  int64_t xoff[4];
  const float* aptr[JB];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = threadIdx.x + 256 * k;
    if (L == 1) {
      xi[k] = e % 16;
      xp[k] = e / 16;
    } else {
      xp[k] = e % 64;
      xi[k] = e / 64;
    }
    const int64_t p = p0 + xp[k];
    xoff[k] = -1;
    if (p < P) {
      int64_t l, h;
      if (P < (int64_t(1) << 31)) {  // 32-bit division where the column index fits (the common case)
        const uint32_t p32 = static_cast<uint32_t>(p), L32 = static_cast<uint32_t>(L);
        h = p32 / L32;
        l = p32 - static_cast<uint32_t>(h) * L32;
      } else {
        l = p % L;
        h = p / L;
      }
      xoff[k] = l + L * I * h;
    }
  }
#pragma unroll
  for (int k = 0; k < JB; ++k) {
    const int e = threadIdx.x + 256 * k;
    ai[k] = e % 16;
    aj[k] = e / 16;
    const int j = j0 + aj[k];
    aptr[k] = j < J ? A + j * sj : nullptr;
  }
  float xr[4], ar[JB];
  auto fetch = [&](int64_t i0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = i0 + xi[k];
      xr[k] = (xoff[k] >= 0 && i < I) ? __ldg(X + xoff[k] + L * i) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < JB; ++k) {
      const int64_t ia = i0 + ai[k];
      ar[k] = (aptr[k] && ia < I) ? __ldg(aptr[k] + ia * si) : 0.f;
    }
  };
  float acc[4][JB];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < JB; ++b) acc[a][b] = 0.f;
  fetch(0);
  for (int64_t i0 = 0; i0 < I; i0 += 16) {
#pragma unroll
    for (int k = 0; k < 4; ++k) Xs[xi[k]][xp[k]] = xr[k];
#pragma unroll
    for (int k = 0; k < JB; ++k) As[ai[k]][aj[k]] = ar[k];
    __syncthreads();
    if (i0 + 16 < I) fetch(i0 + 16);
#pragma unroll
    for (int ii = 0; ii < 16; ++ii) {
      float xv[4], av[JB];
#pragma unroll
      for (int a = 0; a < 4; ++a) xv[a] = Xs[ii][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < JB; ++b) av[b] = As[ii][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < JB; ++b) acc[a][b] = fmaf(xv[a], av[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t p = p0 + tx + 16 * a;
    if (p >= P) continue;
    int64_t l, h;
    if (P < (int64_t(1) << 31)) {
      const uint32_t p32 = static_cast<uint32_t>(p), L32 = static_cast<uint32_t>(L);
      h = p32 / L32;
      l = p32 - static_cast<uint32_t>(h) * L32;
    } else {
      l = p % L;
      h = p / L;
    }
#pragma unroll
    for (int b = 0; b < JB; ++b) {
      const int j = j0 + ty + 16 * b;
      if (j < J) Y[l + L * (j + static_cast<int64_t>(J) * h)] = acc[a][b];
    }
  }
}

// Mode-0 TTM, 4 x NB register tiles (L == 1, I % 4 == 0, 16-byte aligned X, J <= 64).  Block = 256
// columns h x all J rows, 8 warps: warp w owns the row group g = w & 3 (rows g*NB + b, b < NB =
// ceil(J/4)) and the column half hw = w >> 2; lane l owns the 4 adjacent columns hw*128 + 4l + {0..3}.
// Per i a thread does one LDS.128 of X and ceil(NB/4) warp-uniform vector loads of A for 4*NB FMAs:
// FMA-bound, with registers for two blocks per SM.  i advances in steps of 16 (four lanes read one
// column's 64 contiguous bytes), stored transposed into Xs[i][h ^ 8*((i/4)%4)] (XOR swizzle: conflict-
// free transposing stores, contiguous float4 reads); the next step is prefetched into registers.  The
// output tile is staged as Ys[j][h] and written as the contiguous range Y[J*h0, J*(h0+256)).
constexpr int kQCols = 256, kQK = 16, kQXP = kQCols, kQYP = kQCols + 4;
template <int NB>
__global__ void __launch_bounds__(256, NB <= 5 ? 3 : 2) ttm_mode0q_kernel(const float* __restrict__ X, int64_t I, int64_t H,
                                                            const float* __restrict__ A, int J, int64_t sj,
                                                            int64_t si, float* __restrict__ Y) {
  extern __shared__ __align__(16) float m0q[];
  float* Xs = m0q;                // [kQK][kQXP]
  float* As = m0q + kQK * kQXP;   // [kQK][64]: row ii, slot g*16 + b
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp & 3, hw = warp >> 2;
  const int64_t h0 = static_cast<int64_t>(blockIdx.x) * kQCols;
  const int lq = tid & 3;
  const int64_t hbase = h0 + (tid >> 2);
  const float* xcol0 = X + hbase * I + 4 * lq;
  const int64_t col64 = 64 * I;
  const int64_t nv64 = H > hbase ? (H - hbase + 63) / 64 : 0;
  const int nvalid = nv64 < 4 ? static_cast<int>(nv64) : 4;
  float4 xr[4];
  float ar[4];
  auto fetch = [&](int64_t i0) {
    const float* xp = xcol0 + i0;
    const bool iin = i0 + 4 * lq < I;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      xr[k] = (iin && k < nvalid) ? __ldg(reinterpret_cast<const float4*>(xp)) : make_float4(0.f, 0.f, 0.f, 0.f);
      xp += col64;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // A slot e = tid + 256 k: ii = e >> 6, (g', b) = e & 63
      const int e = tid + 256 * k, ii = e >> 6, slot = e & 63, gg = slot >> 4, b = slot & 15;
      const int j = gg * NB + b;
      const int64_t i = i0 + ii;
      ar[k] = (b < NB && j < J && i < I) ? __ldg(A + j * sj + i * si) : 0.f;
    }
  };
  float acc[4][NB];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[c][b] = 0.f;
  fetch(0);
  const int xcol = hw * 128 + 4 * lane;
  const float* as_row = As + g * 16;
  for (int64_t i0 = 0; i0 < I; i0 += kQK) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int hl = ((tid >> 2) + 64 * k) ^ (8 * lq);
      Xs[(4 * lq + 0) * kQXP + hl] = xr[k].x;
      Xs[(4 * lq + 1) * kQXP + hl] = xr[k].y;
      Xs[(4 * lq + 2) * kQXP + hl] = xr[k].z;
      Xs[(4 * lq + 3) * kQXP + hl] = xr[k].w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) As[tid + 256 * k] = ar[k];
    __syncthreads();
    if (i0 + kQK < I) fetch(i0 + kQK);
#pragma unroll 2
    for (int ii = 0; ii < kQK; ++ii) {
      const float4 xv = *reinterpret_cast<const float4*>(Xs + ii * kQXP + (xcol ^ (8 * ((ii >> 2) & 3))));
      float av[(NB + 3) / 4 * 4];
#pragma unroll
      for (int b4 = 0; b4 < (NB + 3) / 4; ++b4) {
        const float4 a = *reinterpret_cast<const float4*>(as_row + ii * 64 + 4 * b4);
        av[4 * b4] = a.x, av[4 * b4 + 1] = a.y, av[4 * b4 + 2] = a.z, av[4 * b4 + 3] = a.w;
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        acc[0][b] = fmaf(xv.x, av[b], acc[0][b]);
        acc[1][b] = fmaf(xv.y, av[b], acc[1][b]);
        acc[2][b] = fmaf(xv.z, av[b], acc[2][b]);
        acc[3][b] = fmaf(xv.w, av[b], acc[3][b]);
      }
    }
    __syncthreads();
  }
  float* Ys = m0q;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = g * NB + b;
    if (j < J)
      *reinterpret_cast<float4*>(Ys + j * kQYP + xcol) = make_float4(acc[0][b], acc[1][b], acc[2][b], acc[3][b]);
  }
  __syncthreads();
  const int64_t ncols = min(static_cast<int64_t>(kQCols), H - h0);
  const int total = static_cast<int>(ncols) * J;
  float* out = Y + h0 * J;
  // e = h * J + j advanced by 256 per step without a division per element
  int h = tid / J, j = tid - (tid / J) * J;
  const int dh = 256 / J, dj = 256 - dh * J;
  for (int e = tid; e < total; e += 256) {
    out[e] = Ys[j * kQYP + h];
    h += dh;
    j += dj;
    if (j >= J) {
      j -= J;
      ++h;
    }
  }
}

size_t ttm_mode0q_smem(int J) {
  const size_t tiles = (static_cast<size_t>(kQK) * kQXP + kQK * 64) * sizeof(float);
  const size_t out = static_cast<size_t>(J) * kQYP * sizeof(float);
  return tiles > out ? tiles : out;
}

template <int NB>
int launch_ttm_mode0q(const float* X, int64_t I, int64_t H, const float* A, int J, int64_t sj, int64_t si, float* Y,
                      cudaStream_t s) {
  KRP_CHECK_CUDA(cudaFuncSetAttribute(ttm_mode0q_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(ttm_mode0q_smem(64))));  // per device: set every call
  const unsigned nb = static_cast<unsigned>((H + kQCols - 1) / kQCols);
  ttm_mode0q_kernel<NB><<<nb, 256, ttm_mode0q_smem(J), s>>>(X, I, H, A, J, sj, si, Y);
  KRP_CHECK_LAUNCH();
  return KRP_OK;
}

// ------------------------------------------------------------------ mode-n Gram
// H[a][b] = sum over fibers f=(l,h) of T[l + L(a + J h)] T[l + L(b + J h)], fp64.
// Fibers come in chunks of 32, converted to fp64 once into shared memory.  Thread blk of a group owns the
// 4 x 4 block (a in 4ta.., b in 4tb..) of H, upper block triangle only (ta <= tb; H is symmetric and the
// lower blocks are mirrored at the end): per fiber it reads 4 + 4 doubles (two LDS.128 each) for 16 DFMAs.
// Several groups (up to 8) split each chunk's fibers (fiber ff goes to group ff % G) and are summed in
// group order at the end, so the result is deterministic for a given plan.
constexpr int kMgPitch = kGramMaxR + 2;  // doubles; 16-byte aligned rows
__global__ void __launch_bounds__(256) mode_gram_partial_kernel(const float* __restrict__ T, int64_t L, int J,
                                                                int64_t H, int64_t fibers_per_block,
                                                                double* __restrict__ partial) {
  __shared__ __align__(16) double F[32][kMgPitch];
  __shared__ double red[3456];  // (G - 1) * T2 * 16 <= 3456 for every J <= 64
  const int tid = threadIdx.x;
  const int nblk = (J + 3) >> 2, T2 = nblk * (nblk + 1) / 2;
  int G = 256 / T2;
  G = G < 1 ? 1 : (G > 8 ? 8 : G);
  const int g = tid / T2, blk = tid - g * T2;
  const bool active = g < G;
  int ta = 0, tb = blk;  // blk -> (ta, tb), ta <= tb, row-major over the upper block triangle
  while (tb >= nblk - ta) {
    tb -= nblk - ta;
    ++ta;
  }
  tb += ta;
  const int Jp = nblk * 4;
  const int64_t nf = L * H;
  const int64_t f_begin = static_cast<int64_t>(blockIdx.x) * fibers_per_block;
  const int64_t f_end = min(nf, f_begin + fibers_per_block);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t fb = f_begin; fb < f_end; fb += 32) {
    const int64_t rem = f_end - fb;
    const int nff = rem < 32 ? static_cast<int>(rem) : 32;
    if (L == 1) {  // the chunk is the contiguous range T[J fb, J (fb + nff))
      const float* src = T + J * fb;
      for (int e = tid; e < 32 * Jp; e += 256) {
        const int ff = e / Jp, a = e - ff * Jp;
        F[ff][a] = (ff < nff && a < J) ? static_cast<double>(__ldg(src + ff * J + a)) : 0.0;
      }
    } else {  // ff = tid % 32 is fixed per thread: one (l, h) decomposition per chunk
      const int ff = tid & 31;
      const int64_t f = fb + ff;
      const int64_t l = f % L, h = f / L;
      const float* src = T + l + L * J * h;
      for (int a = tid >> 5; a < Jp; a += 8)
        F[ff][a] = (ff < nff && a < J) ? static_cast<double>(__ldg(src + L * a)) : 0.0;
    }
    __syncthreads();
    if (active) {
      for (int ff = g; ff < nff; ff += G) {
        const double2 a01 = *reinterpret_cast<const double2*>(&F[ff][4 * ta]);
        const double2 a23 = *reinterpret_cast<const double2*>(&F[ff][4 * ta + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&F[ff][4 * tb]);
        const double2 b23 = *reinterpret_cast<const double2*>(&F[ff][4 * tb + 2]);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
  if (active && g > 0)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[((g - 1) * T2 + blk) * 16 + i * 4 + j] = acc[i][j];
  __syncthreads();
  if (active && g == 0) {
    for (int gg = 1; gg < G; ++gg)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += red[((gg - 1) * T2 + blk) * 16 + i * 4 + j];
    double* out = partial + static_cast<int64_t>(blockIdx.x) * J * J;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ra = 4 * ta + i, cb = 4 * tb + j;
        if (ra < J && cb < J) {
          out[ra * J + cb] = acc[i][j];
          out[cb * J + ra] = acc[i][j];
        }
      }
  }
}

struct MGPlan {
  int P;
  int64_t per_block;
};
MGPlan plan_mode_gram(const Dims& g, int n) {
  const int64_t nf = g.N / g.n[n];
  MGPlan p;
  int64_t P = (nf + 31) / 32;  // one 32-fiber tile per block while that fills up to 592 blocks
  if (P > 592) P = 592;
  if (P < 1) P = 1;
  p.per_block = ((nf + P - 1) / P + 31) / 32 * 32;
  p.P = static_cast<int>((nf + p.per_block - 1) / p.per_block);
  if (p.P < 1) p.P = 1;
  return p;
}

// ------------------------------------------------------------------ symmetric eigensolver (Jacobi)
// One-sided (Hestenes) cyclic Jacobi on the symmetric PSD Gram matrix H: right rotations A <- A J (A = H
// initially) until the columns of A = H V are mutually orthogonal; then H V = V Λ, so ||a_i|| = λ_i and
// v_i = a_i / λ_i: V itself is never formed (the rounds are bound by shared-memory traffic, which this
// halves).  Round-robin pairing (m-1 rounds of m/2 disjoint pairs per
// sweep, tabulated in shared memory once); ONE HALF-WARP PER PAIR: 16 lanes hold columns p, q of A and V
// (rows l, l+16, l+32, l+48 per lane: each half-warp access is one conflict-free 128-byte wavefront),
// form γ = a_p·a_q by an xor-butterfly reduction (all 16 lanes end with bit-identical sums, so they form
// the same rotation) and take α = ||a_p||^2, β = ||a_q||^2 from norms kept in shared memory (recomputed
// exactly at every sweep start, updated by α' = c²α - 2csγ + s²β, β' = s²α + 2csγ + c²β after a rotation),
// rotate, and write the columns back in place (a round's pairs are disjoint: no double buffer).  One named
// barrier per round.  The round is issue-bound
// (the SM runs m/4 warps of ~160 instructions each), so the rotation uses fast fp32 approximations for the
// ANGLE only; (c, s) are renormalised in fp64 (c^2 + s^2 = 1 to fp64 rounding), so every update is an
// exact-to-rounding orthogonal rotation and V stays orthogonal; an approximate angle leaves γ' ~ 1e-6 γ,
// which the next sweep removes.  A pair is rotated while γ^2 > (1e-13)^2 αβ (above the ~m·u rounding
// floor of the dot products); the sweep loop ends after a sweep without rotations.
__device__ __forceinline__ void jacobi_pair(int round, int k, int m, int& p, int& q) {
  int a, b;
  if (k == 0) {
    a = m - 1;
    b = round;
  } else {
    a = (round + k) % (m - 1);
    b = (round - k + (m - 1)) % (m - 1);
  }
  p = a < b ? a : b;
  q = a < b ? b : a;
}

// (c, s) of the rotation orthogonalising columns with Gram [[α, γ], [γ, β]]: t = sign(x) y / (|x| +
// sqrt(x^2 + y^2)) with x = β - α, y = 2γ (sign(0) = +1), c = 1 / sqrt(1 + t^2), s = t c; the pair is
// then a_p' = c a_p - s a_q, a_q' = s a_p + c a_q.
__device__ __forceinline__ double rsqrt_approx_f64(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double rcp_approx_f64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ void jacobi_rot(double alpha, double beta, double gamma, double& c, double& s) {
  const double x = beta - alpha, y = 2.0 * gamma;
  // the angle from the hardware's approximate fp64 reciprocal / reciprocal square root (~20 bits; full fp64
  // range, so no scaling is needed)
  const double r2 = fma(x, x, y * y);
  const double t = (x >= 0.0 ? y : -y) * rcp_approx_f64(fabs(x) + r2 * rsqrt_approx_f64(r2));
  double cd = rsqrt_approx_f64(fma(t, t, 1.0)), sd = t * cd;
  // two Newton steps for 1/sqrt(n), n = c^2 + s^2 = 1 + O(1e-6): |c^2 + s^2 - 1| -> O(1e-16)
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double n = fma(cd, cd, sd * sd);
    const double f = fma(-0.5, n, 1.5);
    cd *= f;
    sd *= f;
  }
  c = cd;
  s = sd;
}

__device__ __forceinline__ double halfwarp_sum_f64(double v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct EigBatch {
  const double* H[kMaxD];
  float* U[kMaxD];
  int r[kMaxD];
};

// one problem per block (blockIdx.x selects (H, r, U) of the batch); columns stored contiguously:
// A[j * 64 + i] = a_j(i), V likewise, rows >= J zero
__global__ void __launch_bounds__(1024) jacobi_top_kernel(EigBatch batch, int J) {
  const double* __restrict__ Hm = batch.H[blockIdx.x];
  float* __restrict__ U = batch.U[blockIdx.x];
  const int r = batch.r[blockIdx.x];
  extern __shared__ double dyn_smem[];
  double* A = dyn_smem;                  // [64][64]
  double* V = dyn_smem + 64 * 64;        // [64][64]
  __shared__ uint16_t ptab[kGramMaxR - 1][kGramMaxR / 2];  // round-robin pairs: p | q << 8
  __shared__ double lam[kGramMaxR];
  __shared__ double cn[kGramMaxR];  // ||a_j||^2: exact at each sweep start, updated by the rotation formulas
  __shared__ int order[kGramMaxR];
  __shared__ int rotated[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = J + (J & 1);  // even number of players; column J (if odd J) is a zero dummy
  const int half = m / 2;
  const int nwork = (half + 1) / 2;  // warps with a pair in either half
  for (int e = tid; e < (m - 1) * half; e += blockDim.x) {
    int p, q;
    jacobi_pair(e / half, e % half, m, p, q);
    ptab[e / half][e % half] = static_cast<uint16_t>(p | (q << 8));
  }
  for (int e = tid; e < 64 * 64; e += blockDim.x) {
    const int j = e >> 6, i = e & 63;
    A[e] = (i < J && j < J) ? Hm[i * J + j] : 0.0;  // H symmetric: column j = row j
  }
  if (tid < 2) rotated[tid] = 0;
  __syncthreads();
  const int k = 2 * warp + (lane >> 4);  // this half-warp's pair slot
  const int l = lane & 15;
#ifdef KRP_DEV_TRACE
  int dev_sweeps = 0;
  long long dv_t0 = clock64(), dv_red = 0, dv_rot = 0, dv_bar = 0, dv_rounds = 0;
#endif
  for (int sweep = 0; sweep < 30 && m >= 2; ++sweep) {
#ifdef KRP_DEV_TRACE
    dev_sweeps = sweep + 1;
#endif
    const int flag = sweep & 1;  // rotated[flag] collects this sweep; rotated[flag ^ 1] is reset for the next
    for (int j = warp; j < m; j += blockDim.x >> 5) {  // exact column norms (fixed-order warp sums)
      const double a0 = A[j * 64 + lane], a1 = A[j * 64 + lane + 32];
      const double n2 = warp_sum_f64(fma(a0, a0, a1 * a1));
      if (lane == 0) cn[j] = n2;
    }
    __syncthreads();
    if (warp < nwork) {
      const bool act = k < half;
      int pq = act ? ptab[0][k] : 0;
      double vc = 1.0, vs = 0.0;
      for (int round = 0; round < m - 1; ++round) {
#ifdef KRP_DEV_TRACE
        const long long c0 = clock64();
#endif
        double* ap = A + (pq & 0xFF) * 64 + l;
        double* aq = A + (pq >> 8) * 64 + l;
        double pv[4], qv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          pv[t] = act ? ap[16 * t] : 0.0;
          qv[t] = act ? aq[16 * t] : 0.0;
        }
        // α, β: the tracked column norms (a sweep without rotations keeps them exact, so the stopping test is
        // exact); γ: a 16-lane butterfly
        const double al = act ? cn[pq & 0xFF] : 0.0, be = act ? cn[pq >> 8] : 0.0;
        double ga = 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) ga = fma(pv[t], qv[t], ga);
        ga = halfwarp_sum_f64(ga);
#ifdef KRP_DEV_TRACE
        const long long c1 = clock64();
#endif
        if (act && ga * ga > 1e-26 * (al * be)) {  // uniform within the half-warp
          jacobi_rot(al, be, ga, vc, vs);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            ap[16 * t] = vc * pv[t] - vs * qv[t];
            aq[16 * t] = vs * pv[t] + vc * qv[t];
          }
          if (l == 0) {
            rotated[flag] = 1;
            const double cc = vc * vc, ss = vs * vs, cs2 = 2.0 * vc * vs * ga;
            cn[pq & 0xFF] = fma(cc, al, fma(ss, be, -cs2));
            cn[pq >> 8] = fma(ss, al, fma(cc, be, cs2));
          }
        }
        const int next = (act && round + 1 < m - 1) ? ptab[round + 1][k] : 0;
        // all pairs of this round are done before the next round re-pairs the columns
#ifdef KRP_DEV_TRACE
        const long long c2 = clock64();
#endif
        asm volatile("bar.sync 1, %0;" ::"r"(nwork * 32) : "memory");
#ifdef KRP_DEV_TRACE
        const long long c3 = clock64();
        dv_red += c1 - c0;
        dv_rot += c2 - c1;
        dv_bar += c3 - c2;
        ++dv_rounds;
#endif
        pq = next;
      }
    }
    __syncthreads();
    const bool again = rotated[flag] != 0;
    if (tid == 0) rotated[flag ^ 1] = 0;
    __syncthreads();
    if (!again) break;
  }
#ifdef KRP_DEV_TRACE
  if (tid == 0)
    printf("jacobi block %d J=%d: %d sweeps, %lld rounds, %lld cycles total; per round: red %lld rot %lld bar %lld\n",
           blockIdx.x, J, dev_sweeps, dv_rounds, clock64() - dv_t0, dv_red / max(dv_rounds, 1LL),
           dv_rot / max(dv_rounds, 1LL), dv_bar / max(dv_rounds, 1LL));
#endif
  // λ_j = ||a_j|| (fixed-order warp sums), then the r largest, descending
  for (int j = warp; j < J; j += blockDim.x >> 5) {
    const double a0 = A[j * 64 + lane], a1 = A[j * 64 + lane + 32];
    const double n2 = warp_sum_f64(fma(a0, a0, a1 * a1));
    if (lane == 0) lam[j] = sqrt(n2);
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < J; ++i) order[i] = i;
    for (int t = 0; t < r; ++t) {
      int best = t;
      for (int i = t + 1; i < J; ++i)
        if (lam[order[i]] > lam[order[best]]) best = i;
      const int tmp = order[t];
      order[t] = order[best];
      order[best] = tmp;
    }
  }
  __syncthreads();
  // eigenvectors v_t = a_t / λ_t (H V = V Λ).  The converged columns are pairwise orthogonal RELATIVE to
  // their own norms, however small (noise-level λ included), so a_t / λ_t is orthonormal; only a column
  // that is exactly zero (or underflows: λ_t <= 1e-150 λ_max; r > rank H) gets a unit vector orthogonalised
  // against the others instead (serial, rare)
  double* Uf = V;  // [r][64]
  const double thr = 1e-150 * lam[order[0]];
  for (int e = tid; e < r * 64; e += blockDim.x) {
    const int t = e >> 6, i = e & 63;
    const double lt = lam[order[t]];
    Uf[e] = (i < J && lt > thr) ? A[order[t] * 64 + i] / lt : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    for (int t = 0; t < r; ++t) {
      if (lam[order[t]] > thr) continue;
      for (int j = 0; j < J; ++j) {
        double* v = Uf + t * 64;
        for (int i = 0; i < J; ++i) v[i] = (i == j) ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
          for (int u = 0; u < r; ++u) {
            if (u == t) continue;
            const double* w = Uf + u * 64;
            double dp = 0.0;
            for (int i = 0; i < J; ++i) dp = fma(w[i], v[i], dp);
            for (int i = 0; i < J; ++i) v[i] = fma(-dp, w[i], v[i]);
          }
        double nn = 0.0;
        for (int i = 0; i < J; ++i) nn = fma(v[i], v[i], nn);
        if (nn > 0.25) {
          const double inv = 1.0 / sqrt(nn);
          for (int i = 0; i < J; ++i) v[i] *= inv;
          break;
        }
      }
    }
  }
  __syncthreads();
  // canonical signs (reading R24): each eigenvector's entry of largest magnitude (first on ties) positive
  for (int t = tid; t < r; t += blockDim.x) {
    const double* v = Uf + t * 64;
    int best = 0;
    for (int i = 1; i < J; ++i)
      if (fabs(v[i]) > fabs(v[best])) best = i;
    lam[t] = v[best] < 0.0 ? -1.0 : 1.0;  // lam (read above) is reused for the signs
  }
  __syncthreads();
  for (int e = tid; e < J * r; e += blockDim.x) {
    const int i = e / r, t = e % r;
    U[e] = static_cast<float>(lam[t] * Uf[t * 64 + i]);
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
  chol_inv_kernel<<<1, kCholThreads, 0, s>>>(G, R, rows, Li, flag_dev, 1);
  KRP_CHECK_LAUNCH();
  apply_linv_kernel<float><<<nb, 256, 0, s>>>(Y, rows, R, Li, Q1, nullptr);
  KRP_CHECK_LAUNCH();
  // pass 2
  KRP_TRY(gram<double>(Q1, rows, R, G, part, s));
  chol_inv_kernel<<<1, kCholThreads, 0, s>>>(G, R, rows, Li, flag_dev, 0);
  KRP_CHECK_LAUNCH();
  apply_linv_kernel<double><<<nb, 256, 0, s>>>(Q1, rows, R, Li, Q2, nullptr);
  KRP_CHECK_LAUNCH();
  // pass 3 (restores orthogonality after a shifted first pass; skipped on the device otherwise, so the
  // unshifted case is plain CholeskyQR2 and the last apply is an exact copy through Linv = I)
  KRP_TRY(gram<double>(Q2, rows, R, G, part, s, flag_dev));
  chol_inv_kernel<<<1, kCholThreads, 0, s>>>(G, R, rows, Li, flag_dev, 2);
  KRP_CHECK_LAUNCH();
  apply_linv_kernel<double><<<nb, 256, 0, s>>>(Q2, rows, R, Li, Qd, Qf);
  KRP_CHECK_LAUNCH();
  ar.off = mark;
  return KRP_OK;
}

int sum_partials_f64(const double* partial, int P, int64_t len, double* out, cudaStream_t s) {
  sum_partials_f64_kernel<<<static_cast<unsigned>((len + 31) / 32), 1024, 0, s>>>(partial, P, len, out);
  KRP_CHECK_LAUNCH();
  return KRP_OK;
}

size_t ttm_ws_bytes(const Dims& g, int n, int J) {
  return (n == 0 && J >= 1 && J <= 64 && g.n[0] % 4 == 0) ? ttm0_tc_ws_bytes(g.n[0], J) : 0;
}

int ttm(const float* X, const Dims& g, int n, const float* A, int J, int64_t sj, int64_t si, float* Y,
        cudaStream_t s, Arena* ar) {
  const int64_t L = g.stride[n], I = g.n[n], H = g.N / (L * I);
  const int64_t P = L * H;
  if (P == 0 || J == 0) return KRP_OK;
  if (ar && L == 1 && ttm0_tc_ok(X, I, H, J) && (ar->cap - ar->off) >= ttm0_tc_ws_bytes(I, J))
    return ttm0_tc(X, I, H, A, J, sj, si, Y, *ar, s);
  if (L == 1 && J <= 64 && I % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && H >= 148 * kQCols / 8) {
    switch ((J + 3) / 4) {
      case 1: return launch_ttm_mode0q<1>(X, I, H, A, J, sj, si, Y, s);
      case 2: return launch_ttm_mode0q<2>(X, I, H, A, J, sj, si, Y, s);
      case 3: return launch_ttm_mode0q<3>(X, I, H, A, J, sj, si, Y, s);
      case 4: return launch_ttm_mode0q<4>(X, I, H, A, J, sj, si, Y, s);
      case 5: return launch_ttm_mode0q<5>(X, I, H, A, J, sj, si, Y, s);
      case 6: return launch_ttm_mode0q<6>(X, I, H, A, J, sj, si, Y, s);
      case 7: return launch_ttm_mode0q<7>(X, I, H, A, J, sj, si, Y, s);
      case 8: return launch_ttm_mode0q<8>(X, I, H, A, J, sj, si, Y, s);
      case 9: return launch_ttm_mode0q<9>(X, I, H, A, J, sj, si, Y, s);
      case 10: return launch_ttm_mode0q<10>(X, I, H, A, J, sj, si, Y, s);
      case 11: return launch_ttm_mode0q<11>(X, I, H, A, J, sj, si, Y, s);
      case 12: return launch_ttm_mode0q<12>(X, I, H, A, J, sj, si, Y, s);
      case 13: return launch_ttm_mode0q<13>(X, I, H, A, J, sj, si, Y, s);
      case 14: return launch_ttm_mode0q<14>(X, I, H, A, J, sj, si, Y, s);
      case 15: return launch_ttm_mode0q<15>(X, I, H, A, J, sj, si, Y, s);
      default: return launch_ttm_mode0q<16>(X, I, H, A, J, sj, si, Y, s);
    }
  }
  const unsigned nb = static_cast<unsigned>((P + 63) / 64);
  const int jb = J >= 64 ? 4 : (J + 15) / 16;  // j tile 16 jb: no more than 15 padded j per launch
  for (int j0 = 0; j0 < J; j0 += 16 * jb) {
    switch (jb) {
      case 1: ttm_kernel<1><<<nb, 256, 0, s>>>(X, L, I, H, A, J, sj, si, Y, j0); break;
      case 2: ttm_kernel<2><<<nb, 256, 0, s>>>(X, L, I, H, A, J, sj, si, Y, j0); break;
      case 3: ttm_kernel<3><<<nb, 256, 0, s>>>(X, L, I, H, A, J, sj, si, Y, j0); break;
      default: ttm_kernel<4><<<nb, 256, 0, s>>>(X, L, I, H, A, J, sj, si, Y, j0); break;
    }
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
  sum_partials_f64_kernel<<<static_cast<unsigned>((len + 31) / 32), 1024, 0, s>>>(part, p.P, len, H);
  KRP_CHECK_LAUNCH();
  ar.off = mark;
  return KRP_OK;
}

int sym_eig_top_batched(const double* const* H, int count, int J, const int* r, float* const* U, cudaStream_t s) {
  if (count < 1 || count > kMaxD || J > kGramMaxR) {
    set_error("eigensolver: count=%d J=%d unsupported", count, J);
    return KRP_EINVAL;
  }
  EigBatch b{};
  for (int k = 0; k < count; ++k) {
    if (r[k] > J || r[k] < 0) {
      set_error("eigensolver: J=%d r=%d unsupported", J, r[k]);
      return KRP_EINVAL;
    }
    b.H[k] = H[k];
    b.U[k] = U[k];
    b.r[k] = r[k];
  }
  KRP_TRY(set_square_smem_attrs());
  jacobi_top_kernel<<<count, 1024, kJacobiSmem, s>>>(b, J);
  KRP_CHECK_LAUNCH();
  return KRP_OK;
}

int sym_eig_top(const double* H, int J, int r, float* U, cudaStream_t s) {
  return sym_eig_top_batched(&H, 1, J, &r, &U, s);
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
