// Roofline denominators that MEASURED_PEAKS.json does not carry: FP64 DFMA
// throughput and shared-memory LDS.128 bandwidth, measured on the current
// device (the FSE kernel is FP64/shared-memory bound, not HBM/tensor bound).
#include <cuda_runtime.h>

#include "fse_kernels.cuh"
#include "host_internal.hpp"

namespace {

constexpr int kChains = 8;

__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
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

// FP64 tensor-core path (mma.sync m8n8k4 .f64; tcgen05 has no f64 kind): the FP64 datapath's
// measured maximum (DFMA and DMMA share it, profiles/r1_dmma_bench.txt)
__global__ void dmma_peak_kernel(double* out, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[kChains][2];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void lds_peak_kernel(double* out, int iters) {
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

}  // namespace

// DMMA m8n8k4: 8 x 8 x 4 MACs = 512 flops per warp instruction
extern "C" int tf_calibrate_peaks(int device, double* dfma_tflops, double* dmma_tflops, double* smem_tbs) {
  int rc = tf_calibrate(device, dfma_tflops, smem_tbs);
  if (rc != TF_OK) return rc;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, 64) != cudaSuccess) return tfh::set_error(TF_ENOMEM, "calibrate alloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  const int threads = 128, blocks = sms * 4, iters = 20000;
  for (int rep = 0; rep < 4; ++rep) {
    float ms = 0.f;
    cudaEventRecord(e0);
    dmma_peak_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 512.0 * kChains * iters * (threads / 32) * static_cast<double>(blocks);
    if (rep && fl / (ms * 1e-3) > best) best = fl / (ms * 1e-3);
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return tfh::set_error(TF_ECUDA, cudaGetErrorString(e));
  if (dmma_tflops) *dmma_tflops = best / 1e12;
  return TF_OK;
}

extern "C" int tf_calibrate(int device, double* fp64_tflops, double* smem_tbs) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return tfh::set_error(TF_ECUDA, cudaGetErrorString(e));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, 64) != cudaSuccess) return tfh::set_error(TF_ENOMEM, "calibrate alloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best_fma = 0.0, best_lds = 0.0;
  const int threads = 512, blocks = sms * 4, iters = 20000;
  for (int rep = 0; rep < 4; ++rep) {
    float ms = 0.f;
    cudaEventRecord(e0);
    dfma_peak_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * kChains * iters * static_cast<double>(threads) * blocks;
    if (rep && fl / (ms * 1e-3) > best_fma) best_fma = fl / (ms * 1e-3);
    cudaEventRecord(e0);
    lds_peak_kernel<<<blocks, 256>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double by = 16.0 * 4 * iters * 256.0 * blocks;
    if (rep && by / (ms * 1e-3) > best_lds) best_lds = by / (ms * 1e-3);
  }
  e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return tfh::set_error(TF_ECUDA, cudaGetErrorString(e));
  if (fp64_tflops) *fp64_tflops = best_fma / 1e12;
  if (smem_tbs) *smem_tbs = best_lds / 1e12;
  return TF_OK;
}

// Exactness self-test of the kernel's hoisted-reciprocal division (div_rn)
// against __ddiv_rn on n hashed operand pairs; *mismatches must be 0.
extern "C" int tf_selftest_div(int device, int64_t n, uint64_t seed, int64_t* mismatches) {
  if (!mismatches || n < 0) return tfh::set_error(TF_EINVAL, "bad arguments");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return tfh::set_error(TF_ECUDA, cudaGetErrorString(e));
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return tfh::set_error(TF_ENOMEM, "selftest alloc");
  cudaMemset(d, 0, sizeof(*d));
  e = tfb::div_selftest_launch(n, seed, d, nullptr);
  unsigned long long bad = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&bad, d, sizeof(bad), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return tfh::set_error(TF_ECUDA, cudaGetErrorString(e));
  *mismatches = static_cast<int64_t>(bad);
  return TF_OK;
}
