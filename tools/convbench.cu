// Throughput microbenchmarks (per SM per clock): F2F.F64.F32, DFMA, SHFL, LDS.64/LDS.128.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k_f2f(const float* in, double* out) {
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = in[threadIdx.x + i];
  double acc[8] = {};
#pragma unroll 4
  for (int it = 0; it < N; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i] += (double)f[i];  // F2F + DADD
      f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(const float* in, double* out) {
  double f[8];
  for (int i = 0; i < 8; ++i) f[i] = in[threadIdx.x + i];
  double acc[8] = {};
#pragma unroll 4
  for (int it = 0; it < N; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += f[i]; }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_shfl(const float* in, double* out) {
  int v[8];
  for (int i = 0; i < 8; ++i) v[i] = __float_as_int(in[threadIdx.x + i]);
#pragma unroll 4
  for (int it = 0; it < N; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __shfl_sync(0xffffffffu, v[i], (threadIdx.x + it + i) & 31);
  }
  int s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* in; double* out;
  cudaMalloc(&in, 1 << 20); cudaMalloc(&out, 1 << 24);
  cudaMemset(in, 0, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, void (*k)(const float*, double*), double ops_per_thread_iter) {
    for (int w = 0; w < 2; ++w) k<<<sms * 4, 512>>>(in, out);
    cudaEventRecord(a); k<<<sms * 4, 512>>>(in, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 4 * 512 * N * ops_per_thread_iter;
    double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-8s %8.3f ms  %6.1f lane-ops/clk/SM (at %d MHz max clock)\n", name, ms, per_sm_clk, clk / 1000);
  };
  run("f2f+dadd", k_f2f, 8);
  run("dadd", k_dadd, 8);
  run("shfl", k_shfl, 8);
  return 0;
}
