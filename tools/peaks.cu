// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// FP64 DFMA / DADD throughput and shared-memory LDS.128 bandwidth on this B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
//   ./tools/peaks   -> one JSON line
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dadd_kernel(double* out, int iters, double a) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __dadd_rn(x[c], a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void lds_kernel(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc[4] = {};
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double2 v = buf[(idx + c * 256) & 2047];
      acc[c].x += v.x;
      acc[c].y += v.y;
    }
    idx += 32;
  }
  double s = 0;
  for (int c = 0; c < 4; ++c) s += acc[c].x + acc[c].y;
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  double* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = prop.multiProcessorCount;
  const int threads = 512, blocks = sms * 4;
  float ms;
  double best_fma = 0, best_add = 0, best_lds = 0;
  for (int rep = 0; rep < 5; ++rep) {
    const int iters = 20000;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * kChains * iters * double(threads) * blocks;
    if (rep) best_fma = fl / (ms * 1e-3) > best_fma ? fl / (ms * 1e-3) : best_fma;
    cudaEventRecord(e0);
    dadd_kernel<<<blocks, threads>>>(d, iters, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ad = 1.0 * kChains * iters * double(threads) * blocks;
    if (rep) best_add = ad / (ms * 1e-3) > best_add ? ad / (ms * 1e-3) : best_add;
    const int li = 20000;
    cudaEventRecord(e0);
    lds_kernel<<<blocks, 256>>>(d, li);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double by = 16.0 * 4 * li * 256.0 * blocks;
    if (rep) best_lds = by / (ms * 1e-3) > best_lds ? by / (ms * 1e-3) : best_lds;
  }
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"fp64_fma_tflops\": %.3f, \"fp64_add_tops\": %.3f, \"smem_lds128_tbs\": %.3f, "
         "\"sms\": %d, \"clock_mhz_attr\": %d, \"error\": \"%s\"}\n",
         best_fma / 1e12, best_add / 1e12, best_lds / 1e12, sms, clk_khz / 1000,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
