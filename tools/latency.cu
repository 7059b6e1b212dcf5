// Dependent-chain latency microbenchmarks (one warp): DADD, DMUL, DFMA, LDS.128,
// CREDUX (__reduce_max_sync), SHFL (64-bit), BAR.SYNC (1 and 4 warps), IADD.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency tools/latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void lat(long long* out, double* dsink, unsigned* usink, int n) {
  __shared__ double2 sm[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    sm[i] = make_double2(i, i);
    idx[i] = (i * 7 + 1) & 1023;
  }
  __syncthreads();
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0);
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, 1.0000001);
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0);
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 1.0000001, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0);
  // LDS chain (pointer chasing through idx)
  int p = threadIdx.x & 1023;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = idx[p];
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0);
  // LDS.128 dependent (address from loaded value)
  double2 v = sm[p];
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = sm[(static_cast<int>(v.x) + 1) & 1023];
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0);
  // CREDUX chain
  unsigned u = threadIdx.x + p;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + threadIdx.x) & 0xffff;
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0);
  // SHFL 64-bit chain
  unsigned long long k = threadIdx.x + u;
  t0 = clock64();
  for (int i = 0; i < n; ++i) k = __shfl_xor_sync(0xffffffffu, k, 1) + 1;
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = (t1 - t0);
  // BAR.SYNC
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[7] = (t1 - t0);
  // IADD chain
  int q = threadIdx.x + static_cast<int>(k);
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = q * 3 + 1;
  t1 = clock64();
  if (threadIdx.x == 0) out[8] = (t1 - t0);
  dsink[threadIdx.x] = x + v.x;
  usink[threadIdx.x] = u + q;
}

int main() {
  long long* d;
  double* ds;
  unsigned* us;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaMalloc(&ds, 1024 * 8);
  cudaMalloc(&us, 1024 * 4);
  const char* names[] = {"DADD", "DMUL", "DFMA", "LDS32(chase)", "LDS128(dep)", "CREDUX", "SHFL64",
                         "BAR.SYNC", "IMAD"};
  for (int warps : {1, 4}) {
    lat<<<1, 32 * warps>>>(d, ds, us, N);
    lat<<<1, 32 * warps>>>(d, ds, us, N);
    long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warps=%d:", warps);
    for (int i = 0; i < 9; ++i) printf(" %s=%.1f", names[i], double(h[i]) / N);
    printf("\n");
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
