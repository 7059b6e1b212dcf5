// Per-warp FP64 issue rate: cycles per DFMA for 1..4 warps per SMSP (8 independent chains).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k(double* out, double a, double b, long long* cyc) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < N; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k16(double* out, double a, double b, long long* cyc) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < N; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int wps = 1; wps <= 4; ++wps) {
    for (int v = 0; v < 2; ++v) {
      auto f = v ? k16 : k;
      const int chains = v ? 16 : 8;
      f<<<sms, 128 * wps>>>(out, 1.0000001, 1e-9, cyc);
      f<<<sms, 128 * wps>>>(out, 1.0000001, 1e-9, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("warps/SMSP %d chains %2d: %.2f cycles per warp-DFMA per warp, %.2f per SMSP\n", wps, chains,
             (double)c / (N * chains), (double)c / (N * chains) / wps);
    }
  }
  return 0;
}
