// jacbench.cu — timing / sweep count of the core-truncation Jacobi eigensolver (dev tool; kernel text
// copied from csrc/krp_linalg.cu).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o jacbench jacbench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
constexpr int kGramMaxR = 64;
__global__ void __launch_bounds__(256) jacobi_top_kernel(const double* __restrict__ Hm, int J, int r,
                                                         float* __restrict__ U, int* sweeps_out) {
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
      for (int e = tid; e < J * J; e += blockDim.x) {
        const int i = e / J, j = e % J;
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
    if (!(offn > 1e-26 * totn) || m < 2) { if (tid == 0) *sweeps_out = sweep; break; }
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
      // rows: A <- J^T A
      for (int e = tid; e < (m / 2) * J; e += blockDim.x) {
        const int k = e / J, col = e % J;
        const int p = pp[k], q = qq[k];
        if (q >= J) continue;
        const double c = cs[k], s = sn[k];
        const double ap = A[p][col], aq = A[q][col];
        A[p][col] = c * ap - s * aq;
        A[q][col] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int e = tid; e < (m / 2) * J; e += blockDim.x) {
        const int k = e / J, row = e % J;
        const int p = pp[k], q = qq[k];
        if (q >= J) continue;
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


int main() {
  const int J = 40, r = 30;
  std::mt19937 g(0);
  std::normal_distribution<double> nd;
  std::vector<double> G(J * 1600), H(J * J, 0.0);
  for (int i = 0; i < J; ++i) for (int k = 0; k < 1600; ++k) G[i * 1600 + k] = nd(g) * pow(0.8, i);
  for (int i = 0; i < J; ++i) for (int j = 0; j < J; ++j) { double s = 0; for (int k = 0; k < 1600; ++k) s += G[i*1600+k]*G[j*1600+k]; H[i*J+j] = s; }
  double* dH; float* dU; int* dS;
  cudaMalloc(&dH, J*J*8); cudaMalloc(&dU, J*r*4); cudaMalloc(&dS, 4);
  cudaMemcpy(dH, H.data(), J*J*8, cudaMemcpyHostToDevice);
  cudaMemset(dS, 0xff, 4);
  const size_t smem = 2 * kGramMaxR * (kGramMaxR + 1) * sizeof(double);
  cudaFuncSetAttribute(jacobi_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  jacobi_top_kernel<<<1, 256, smem>>>(dH, J, r, dU, dS);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) jacobi_top_kernel<<<1, 256, smem>>>(dH, J, r, dU, dS);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int sw; cudaMemcpy(&sw, dS, 4, cudaMemcpyDeviceToHost);
  printf("jacobi J=%d: %.1f us per launch, sweeps %d (%s)\n", J, ms * 100, sw, cudaGetErrorString(e));
  return 0;
}
