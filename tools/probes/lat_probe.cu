// Latency probe (dev tool): dependent-chain latencies of fp64 / fp32 ops, 64-bit shuffles and a
// 30-warp named barrier on sm_100a.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double x0, float f0) {
  double x = x0 + threadIdx.x * 1e-9;
  float f = f0 + threadIdx.x * 1e-6f;
  long long t0, t1;
  const int N = 256;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x + 1e-7 * x;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = f / (f + 1.5f);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = sqrtf(f + 1.5f);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { __syncthreads(); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = fmaf(f, 0.9999f, 1e-7f);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) / N;
  __shared__ double sm[1024];
  sm[threadIdx.x] = x;
  __syncthreads();
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { double v = sm[idx]; idx = (int)(v * 0.0) + ((idx + 1) & 1023); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = rsqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[10] = (t1 - t0) / N;
  out[threadIdx.x] = x + f + idx;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 16 * 8);
  const char* names[] = {"dfma", "dadd+dmul(fma)", "dsqrt", "drcp(div)", "fdiv", "fsqrt", "shfl64+dadd", "syncthreads",
                         "ffma", "lds64", "drsqrt"};
  for (int nt : {32, 960}) {
    probe<<<1, nt>>>(out, cyc, 1.5, 1.25f);
    cudaDeviceSynchronize();
    printf("threads=%d\n", nt);
    for (int i = 0; i < 11; ++i) printf("  %-16s %lld cycles\n", names[i], cyc[i]);
  }
  return 0;
}
