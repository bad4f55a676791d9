// krp_sketch_simt.cu — fp32 CUDA-core MTTKRP sketch for any shape (the engine for
// shapes the tcgen05 kernel does not tile, e.g. modes shorter than 128, and the
// KRP_ENGINE_SIMT reference engine).
//
//   Y_n(i, r) = sum_c X_(n)(i, c) * prod_{k != n} Omega_k(i_k(c), r)
//
// Grid: (32-row tile of mode n) x (chunk of unfolding columns c).  Each block forms
// the Khatri-Rao rows of 32 columns at a time in shared memory (never in global
// memory), each warp streams a quarter of those columns, per-thread fp32
// accumulators; the 4 warps are combined in a fixed order and every block writes a
// partial I_n x RC tile.  A second kernel sums the partials in fp64, fixed order.
#include <algorithm>

#include "krp_common.cuh"
#include "krp_internal.h"

namespace krp {
namespace {

constexpr int kRowsPerBlock = 32;
constexpr int kColTile = 32;

template <int RC>
__global__ void __launch_bounds__(128) sketch_mode_simt_kernel(const float* __restrict__ X, Dims g, int n,
                                                               OmegaPtrs om, int R, int r0, int64_t ncols,
                                                               int64_t cols_per_chunk, float* __restrict__ partial) {
  __shared__ float kr[kColTile][RC + 1];
  __shared__ float red[4][kRowsPerBlock][RC + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t In = g.n[n], L = g.stride[n];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + lane;
  const int64_t c_begin = static_cast<int64_t>(blockIdx.y) * cols_per_chunk;
  const int64_t c_end = min(ncols, c_begin + cols_per_chunk);
  float acc[RC];
#pragma unroll
  for (int r = 0; r < RC; ++r) acc[r] = 0.f;

  for (int64_t cb = c_begin; cb < c_end; cb += kColTile) {
    // Khatri-Rao rows of columns cb .. cb+31 (other modes in ascending order = column order)
    for (int j = threadIdx.x; j < kColTile * RC; j += blockDim.x) {
      const int cc = j / RC, r = j % RC;
      const int64_t c = cb + cc;
      float prod = 0.f;
      if (c < c_end && r0 + r < R) {
        prod = 1.f;
        int64_t t = c;
        for (int k = 0; k < g.d; ++k) {
          if (k == n) continue;
          const int64_t ik = t % g.n[k];
          t /= g.n[k];
          prod *= __ldg(om.p[k] + ik * R + r0 + r);
        }
      }
      kr[cc][r] = prod;
    }
    __syncthreads();
    if (i < In) {
      for (int cc = w; cc < kColTile; cc += 4) {
        const int64_t c = cb + cc;
        if (c >= c_end) break;
        const int64_t clow = c % L, chigh = c / L;
        const float x = __ldg(X + clow + i * L + chigh * L * In);
#pragma unroll
        for (int r = 0; r < RC; ++r) acc[r] = fmaf(x, kr[cc][r], acc[r]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < RC; ++r) red[w][lane][r] = acc[r];
  __syncthreads();
  // fixed-order combination of the 4 warps; 128 threads write the 32 x RC tile
  for (int j = threadIdx.x; j < kRowsPerBlock * RC; j += blockDim.x) {
    const int row = j / RC, r = j % RC;
    const int64_t ii = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + row;
    if (ii < In) {
      const float s = ((red[0][row][r] + red[1][row][r]) + red[2][row][r]) + red[3][row][r];
      partial[(static_cast<int64_t>(blockIdx.y) * In + ii) * RC + r] = s;
    }
  }
}

__global__ void reduce_partials_kernel(const float* __restrict__ partial, int P, int64_t In, int RC, int R, int r0,
                                       float* __restrict__ Y) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= In * RC) return;
  const int64_t i = idx / RC;
  const int r = static_cast<int>(idx % RC);
  if (r0 + r >= R) return;
  double s = 0.0;
  for (int p = 0; p < P; ++p) s += static_cast<double>(partial[(static_cast<int64_t>(p) * In + i) * RC + r]);
  Y[i * R + r0 + r] = static_cast<float>(s);
}

int rc_for(int R) { return R <= 16 ? 16 : (R <= 32 ? 32 : 64); }

struct SimtPlan {
  int RC, passes, P;
  int64_t ncols, cols_per_chunk, row_tiles;
};

SimtPlan plan_simt(const Dims& g, int n, int R) {
  SimtPlan p;
  p.RC = rc_for(R);
  p.passes = (R + p.RC - 1) / p.RC;
  p.ncols = g.N / g.n[n];
  p.row_tiles = (g.n[n] + kRowsPerBlock - 1) / kRowsPerBlock;
  // aim for ~4 waves of 148 SMs, chunks of at least 256 columns
  int64_t want = (4 * 148 + p.row_tiles - 1) / p.row_tiles;
  int64_t max_chunks = (p.ncols + 255) / 256;
  int64_t P = want < max_chunks ? want : max_chunks;
  if (P < 1) P = 1;
  if (P > 65535) P = 65535;
  p.cols_per_chunk = (p.ncols + P - 1) / P;
  p.cols_per_chunk = (p.cols_per_chunk + kColTile - 1) / kColTile * kColTile;
  p.P = static_cast<int>((p.ncols + p.cols_per_chunk - 1) / p.cols_per_chunk);
  return p;
}

}  // namespace

size_t simt_sketch_ws_bytes(const Dims& g, int n, int R) {
  SimtPlan p = plan_simt(g, n, R);
  return align_up(static_cast<size_t>(p.P) * g.n[n] * p.RC * sizeof(float), 256);
}

int simt_sketch_mode(const float* X, const Dims& g, int n, const OmegaPtrs& om, int R, float* Y, Arena& ar,
                     cudaStream_t s) {
  SimtPlan p = plan_simt(g, n, R);
  size_t mark = ar.off;
  float* partial = ar.take<float>(static_cast<size_t>(p.P) * g.n[n] * p.RC);
  if (ar.overflow()) {
    set_error("workspace too small for the SIMT sketch");
    return KRP_ENOMEM;
  }
  for (int pass = 0; pass < p.passes; ++pass) {
    const int r0 = pass * p.RC;
    dim3 grid(static_cast<unsigned>(p.row_tiles), static_cast<unsigned>(p.P));
    prof_begin(s);
    switch (p.RC) {
      case 16:
        sketch_mode_simt_kernel<16><<<grid, 128, 0, s>>>(X, g, n, om, R, r0, p.ncols, p.cols_per_chunk, partial);
        break;
      case 32:
        sketch_mode_simt_kernel<32><<<grid, 128, 0, s>>>(X, g, n, om, R, r0, p.ncols, p.cols_per_chunk, partial);
        break;
      default:
        sketch_mode_simt_kernel<64><<<grid, 128, 0, s>>>(X, g, n, om, R, r0, p.ncols, p.cols_per_chunk, partial);
        break;
    }
    KRP_CHECK_LAUNCH();
    // algorithmic work of this launch: one read of X, 2*N*RC flops of the single-mode MTTKRP
    prof_end(s, 4.0 * static_cast<double>(g.N), 2.0 * static_cast<double>(g.N) * std::min(p.RC, R - r0));
    const int64_t tot = g.n[n] * p.RC;
    reduce_partials_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(partial, p.P, g.n[n], p.RC, R,
                                                                                     r0, Y);
    KRP_CHECK_LAUNCH();
  }
  ar.off = mark;
  return KRP_OK;
}

}  // namespace krp
