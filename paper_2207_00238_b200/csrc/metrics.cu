// Image-quality metrics on the GPU: the reference's mse, mse_missing,
// psnr and ssim (metrics.hpp:12-90), batched over frames for in-loop parity checks.
//
// Exactness.  The reference accumulates integer-valued squares in binary64
// (metrics.hpp:16-20, 35-40); every partial sum stays below 2^53, so the sums are exact and
// equal to the 64-bit integer sums used here; the final division and log10 run on the host
// with the same expressions -> MSE and PSNR are bit-identical.  SSIM: the five window sums
// of an 8x8 window (metrics.hpp:73-82) are integers (exact in both); the per-window formula
// (metrics.hpp:83-87) is evaluated with the same binary64 operations in the same order
// (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn, no contraction) -> every window value is
// bit-identical; only the order of the final mean's summation differs (fixed-shape tree:
// deterministic, within 1e-12 relative of the reference's sequential sum).
//
// HBM-bound byte work: the SSE kernel streams a, b and the mask once (16-byte loads when
// aligned); the SSIM kernel stages a 128 x (32 + 7) patch of both frames in shared memory and
// slides the 8-row window down each column with integer running sums.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "fse_kernels.cuh"

namespace tfb {

namespace {

constexpr int kSsimTW = 128;  // output windows per CTA row (one thread per column)
constexpr int kSsimTH = 32;   // output window rows per CTA

__device__ __forceinline__ void acc_byte(uint32_t a, uint32_t b, uint32_t k, unsigned long long& sse,
                                         unsigned long long& ssm, unsigned long long& nm) {
  const int d = static_cast<int>(a) - static_cast<int>(b);
  const unsigned long long q = static_cast<unsigned long long>(d * d);
  sse += q;
  if (!k) {
    ssm += q;
    nm += 1;
  }
}

// out[f] = {sum d^2, sum over unknown d^2, unknown count}; known may be null (no mask)
__global__ void __launch_bounds__(256) sse_kernel(const uint8_t* a, const uint8_t* b, const uint8_t* known,
                                                  int64_t n, bool vec, unsigned long long* out) {
  const int f = blockIdx.y;
  const uint8_t* pa = a + static_cast<size_t>(n) * f;
  const uint8_t* pb = b + static_cast<size_t>(n) * f;
  const uint8_t* pk = known ? known + static_cast<size_t>(n) * f : nullptr;
  unsigned long long sse = 0, ssm = 0, nm = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t done = 0;
  if (vec) {  // 16-byte chunks (bases 16-aligned, checked on the host)
    const int64_t nv = n / 16;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv; i += stride) {
      const uint4 va = __ldg(reinterpret_cast<const uint4*>(pa) + i);
      const uint4 vb = __ldg(reinterpret_cast<const uint4*>(pb) + i);
      uint4 vk = make_uint4(~0u, ~0u, ~0u, ~0u);
      if (pk) vk = __ldg(reinterpret_cast<const uint4*>(pk) + i);
      const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w},
                     wk[4] = {vk.x, vk.y, vk.z, vk.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int s = 0; s < 32; s += 8)
          acc_byte((wa[q] >> s) & 255u, (wb[q] >> s) & 255u, (wk[q] >> s) & 255u, sse, ssm, nm);
    }
    done = nv * 16;
  }
  for (int64_t i = done + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    acc_byte(pa[i], pb[i], pk ? pk[i] : 1u, sse, ssm, nm);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
    ssm += __shfl_xor_sync(0xffffffffu, ssm, o);
    nm += __shfl_xor_sync(0xffffffffu, nm, o);
  }
  if ((threadIdx.x & 31) == 0 && (sse | ssm | nm)) {  // integer atomics: order-independent
    atomicAdd(out + 3 * f, sse);
    atomicAdd(out + 3 * f + 1, ssm);
    atomicAdd(out + 3 * f + 2, nm);
  }
}

// Per-CTA partial sums of the window SSIM values of one frame patch:
// kSsimTW output columns x kSsimTH output rows (windows whose top-left corner lies there).
__global__ void __launch_bounds__(kSsimTW) ssim_kernel(const uint8_t* a, const uint8_t* b, int w, int h,
                                                       double c1, double c2, double* partial) {
  constexpr int PW = kSsimTW + 7, PH = kSsimTH + 7;
  __shared__ uint8_t sa[PH][PW + 1], sb[PH][PW + 1];
  __shared__ double red[kSsimTW / 32];
  const int f = blockIdx.z;
  const int x0 = blockIdx.x * kSsimTW, y0 = blockIdx.y * kSsimTH;
  const int nwx = w - 7, nwy = h - 7;  // windows per row / column
  const uint8_t* pa = a + static_cast<size_t>(w) * h * f;
  const uint8_t* pb = b + static_cast<size_t>(w) * h * f;
  for (int i = threadIdx.x; i < PW * PH; i += kSsimTW) {
    const int yy = i / PW, xx = i - yy * PW;
    const int X = x0 + xx, Y = y0 + yy;
    uint8_t va = 0, vb = 0;
    if (X < w && Y < h) {
      const size_t g = static_cast<size_t>(Y) * w + X;
      va = pa[g];
      vb = pb[g];
    }
    sa[yy][xx] = va;
    sb[yy][xx] = vb;
  }
  __syncthreads();
  const int tx = threadIdx.x, wx = x0 + tx;
  const int rows = min(kSsimTH, nwy - y0);
  double total = 0.0;
  if (wx < nwx && rows > 0) {
    // running vertical sums of the horizontal 8-sums: a, b, aa, bb, ab
    int va = 0, vb = 0, vaa = 0, vbb = 0, vab = 0;
    for (int y = 0; y < rows + 7; ++y) {
      int ha = 0, hb = 0, haa = 0, hbb = 0, hab = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int p = sa[y][tx + i], q = sb[y][tx + i];
        ha += p;
        hb += q;
        haa += p * p;
        hbb += q * q;
        hab += p * q;
      }
      va += ha;
      vb += hb;
      vaa += haa;
      vbb += hbb;
      vab += hab;
      if (y >= 8) {  // drop row y - 8
        int ga = 0, gb = 0, gaa = 0, gbb = 0, gab = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int p = sa[y - 8][tx + i], q = sb[y - 8][tx + i];
          ga += p;
          gb += q;
          gaa += p * p;
          gbb += q * q;
          gab += p * q;
        }
        va -= ga;
        vb -= gb;
        vaa -= gaa;
        vbb -= gbb;
        vab -= gab;
      }
      if (y >= 7) {
        // metrics.hpp:83-87, same binary64 operation order (inv_n = 1/64 is exact)
        const double inv_n = 1.0 / 64.0;
        const double mu_a = __dmul_rn(static_cast<double>(va), inv_n);
        const double mu_b = __dmul_rn(static_cast<double>(vb), inv_n);
        const double var_a = __dsub_rn(__dmul_rn(static_cast<double>(vaa), inv_n), __dmul_rn(mu_a, mu_a));
        const double var_b = __dsub_rn(__dmul_rn(static_cast<double>(vbb), inv_n), __dmul_rn(mu_b, mu_b));
        const double cov = __dsub_rn(__dmul_rn(static_cast<double>(vab), inv_n), __dmul_rn(mu_a, mu_b));
        const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_a), mu_b), c1),
                                     __dadd_rn(__dmul_rn(2.0, cov), c2));
        const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu_a, mu_a), __dmul_rn(mu_b, mu_b)), c1),
                                     __dadd_rn(__dadd_rn(var_a, var_b), c2));
        total = __dadd_rn(total, __ddiv_rn(num, den));
      }
    }
  }
  // fixed-shape tree: deterministic for a given frame size
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total = __dadd_rn(total, __shfl_xor_sync(0xffffffffu, total, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = total;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = red[0];
    for (int q = 1; q < kSsimTW / 32; ++q) s = __dadd_rn(s, red[q]);
    partial[(static_cast<size_t>(f) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
  }
}

// out[f] = sum of the frame's n partials (pairwise tree in shared memory, fixed shape)
__global__ void __launch_bounds__(1024) sum_partials_kernel(const double* partial, int n, double* out) {
  __shared__ double s[1024];
  const double* p = partial + static_cast<size_t>(n) * blockIdx.x;
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) t = __dadd_rn(t, p[i]);
  s[threadIdx.x] = t;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] = __dadd_rn(s[threadIdx.x], s[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

}  // namespace

int64_t ssim_partials(int w, int h, int frames) {
  if (w < 8 || h < 8) return 0;
  const int64_t gx = (w - 7 + kSsimTW - 1) / kSsimTW, gy = (h - 7 + kSsimTH - 1) / kSsimTH;
  return gx * gy * frames;
}

cudaError_t quality_launch(const uint8_t* a, const uint8_t* b, const uint8_t* known, int w, int h,
                           int frames, int sms, unsigned long long* sse3, double* partial,
                           double* ssim_sum, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(w) * h;
  cudaError_t e = cudaMemsetAsync(sse3, 0, sizeof(unsigned long long) * 3 * frames, s);
  if (e != cudaSuccess) return e;
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool vec = n % 16 == 0 && al(a) && al(b) && (!known || al(known));
  const int64_t per = vec ? n / 16 : n;
  int gx = static_cast<int>(std::min<int64_t>((per + 255) / 256, static_cast<int64_t>(sms) * 8));
  if (gx < 1) gx = 1;
  sse_kernel<<<dim3(gx, frames), 256, 0, s>>>(a, b, known, n, vec, sse3);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (partial && ssim_sum && w >= 8 && h >= 8) {
    // C1, C2 as the reference spells them (metrics.hpp:68-69), evaluated in binary64
    const double c1 = (0.01 * 255.0) * (0.01 * 255.0);
    const double c2 = (0.03 * 255.0) * (0.03 * 255.0);
    const dim3 grid((w - 7 + kSsimTW - 1) / kSsimTW, (h - 7 + kSsimTH - 1) / kSsimTH, frames);
    ssim_kernel<<<grid, kSsimTW, 0, s>>>(a, b, w, h, c1, c2, partial);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    sum_partials_kernel<<<frames, 1024, 0, s>>>(partial, static_cast<int>(grid.x * grid.y), ssim_sum);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace tfb
