// Diffusion extrapolator (extrapolate.hpp:41-84) on the tile halos of a tiled job, sm_100a.
//
// K Jacobi sweeps: every unknown pixel of a halo takes the mean of its in-bounds 4-neighbours
// (left, right, up, down added in that order, then divided by the count) from the previous
// sweep; known pixels stay fixed; unknown pixels start at 128.  Bit-identical to the
// reference: the same binary64 operations per pixel and sweep (__dadd_rn / __ddiv_rn).
//
// HBM/L2-bound stencil, so sweeps are fused S at a time (temporal blocking): a CTA loads a
// (32 + 2S)^2 window of the current field into shared memory, runs S sweeps there (the valid
// region shrinks by one pixel per sweep) and writes its 32 x 32 patch of the result.  The
// field stays in FP64 in HBM between launches (halo-major, one array per tile).
#include <cuda_runtime.h>

#include <cstdint>

#include "fse_kernels.cuh"

namespace tfb {

namespace {

constexpr int kPatch = 32;

__device__ __forceinline__ int find_tile(const int64_t* poff, int n_tiles, int64_t b) {
  int lo = 0, hi = n_tiles - 1;  // last tile with poff[t] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (poff[mid] <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// cur = known ? pixel : 128 over every halo pixel
__global__ void diffusion_init_kernel(const uint8_t* img, const uint8_t* known, int W, int H,
                                      const TileDesc* tiles, int n_tiles, const int64_t* foff,
                                      double* cur, double* nxt) {
  const int t = blockIdx.y;
  if (t >= n_tiles) return;
  const TileDesc tl = tiles[t];
  const int64_t n = static_cast<int64_t>(tl.hw) * tl.hh;
  const size_t plane = static_cast<size_t>(W) * H * tl.frame;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / tl.hw), x = static_cast<int>(i - static_cast<int64_t>(y) * tl.hw);
    const size_t g = plane + static_cast<size_t>(tl.hy + y) * W + tl.hx + x;
    const double v = known[g] ? static_cast<double>(img[g]) : 128.0;
    cur[foff[t] + i] = v;
    nxt[foff[t] + i] = v;
  }
}

// S fused sweeps: src -> dst for one 32 x 32 patch of one tile halo
template <int S>
__global__ void __launch_bounds__(256) diffusion_sweeps_kernel(const uint8_t* known, int W, int H,
                                                                const TileDesc* tiles, int n_tiles,
                                                                const int64_t* foff, const int64_t* poff,
                                                                const double* src, double* dst,
                                                                int sweeps) {
  constexpr int R = kPatch + 2 * S;  // shared-memory window side
  __shared__ double a[R * R], b[R * R];
  __shared__ uint8_t fl[R * R];  // bit0: inside the halo, bit1: known, bits 2-5: in-bounds L/R/U/D
  const int t = find_tile(poff, n_tiles, blockIdx.x);
  const TileDesc tl = tiles[t];
  const int pw = (tl.hw + kPatch - 1) / kPatch;
  const int p = static_cast<int>(blockIdx.x - poff[t]);
  const int py = p / pw, px = p - py * pw;
  const int x0 = px * kPatch - S, y0 = py * kPatch - S;  // window origin, halo-local
  const size_t plane = static_cast<size_t>(W) * H * tl.frame;
  const double* fs = src + foff[t];
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
    const int wy = i / R, wx = i - wy * R;
    const int x = x0 + wx, y = y0 + wy;
    uint8_t f = 0;
    double v = 0.0;
    if (x >= 0 && x < tl.hw && y >= 0 && y < tl.hh) {
      const size_t g = plane + static_cast<size_t>(tl.hy + y) * W + tl.hx + x;
      f = 1 | (known[g] ? 2 : 0) | (x > 0 ? 4 : 0) | (x + 1 < tl.hw ? 8 : 0) | (y > 0 ? 16 : 0) |
          (y + 1 < tl.hh ? 32 : 0);
      v = fs[static_cast<int64_t>(y) * tl.hw + x];
    }
    fl[i] = f;
    a[i] = v;
    b[i] = v;
  }
  __syncthreads();
  double* cur = a;
  double* nxt = b;
  for (int s = 0; s < sweeps; ++s) {
    const int lo = s + 1, hi = R - 1 - s;  // cells whose neighbours are valid for this sweep
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
      const int wy = i / R, wx = i - wy * R;
      if (wx < lo || wx >= hi || wy < lo || wy >= hi) continue;
      const int f = fl[i];
      if ((f & 3) != 1) continue;  // outside the halo or known: unchanged
      double sum = 0.0;
      int cnt = 0;
      if (f & 4) { sum = __dadd_rn(sum, cur[i - 1]); ++cnt; }
      if (f & 8) { sum = __dadd_rn(sum, cur[i + 1]); ++cnt; }
      if (f & 16) { sum = __dadd_rn(sum, cur[i - R]); ++cnt; }
      if (f & 32) { sum = __dadd_rn(sum, cur[i + R]); ++cnt; }
      // sum / cnt, correctly rounded: exact power-of-two scalings for 1, 2, 4
      double v;
      if (cnt == 4) v = __dmul_rn(sum, 0.25);
      else if (cnt == 2) v = __dmul_rn(sum, 0.5);
      else if (cnt == 1) v = sum;
      else if (cnt == 3) v = __ddiv_rn(sum, 3.0);
      else v = 128.0;
      nxt[i] = v;
    }
    __syncthreads();
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  double* fd = dst + foff[t];
  for (int i = threadIdx.x; i < kPatch * kPatch; i += blockDim.x) {
    const int yy = i / kPatch, xx = i - yy * kPatch;
    const int x = px * kPatch + xx, y = py * kPatch + yy;
    if (x < tl.hw && y < tl.hh) fd[static_cast<int64_t>(y) * tl.hw + x] = cur[(yy + S) * R + xx + S];
  }
}

// unknown core pixels: floor(v + 0.5) clamped to [0, 255] (extrapolate.hpp:75-82)
__global__ void diffusion_final_kernel(const uint8_t* known, uint8_t* out, int W, int H,
                                       const TileDesc* tiles, int n_tiles, const int64_t* foff,
                                       const double* cur) {
  const int t = blockIdx.y;
  if (t >= n_tiles) return;
  const TileDesc tl = tiles[t];
  const int64_t n = static_cast<int64_t>(tl.cw) * tl.ch;
  const size_t plane = static_cast<size_t>(W) * H * tl.frame;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int yy = static_cast<int>(i / tl.cw), xx = static_cast<int>(i - static_cast<int64_t>(yy) * tl.cw);
    const int AX = tl.cx + xx, AY = tl.cy + yy;
    const size_t g = plane + static_cast<size_t>(AY) * W + AX;
    if (known[g]) continue;
    const double v = cur[foff[t] + static_cast<int64_t>(AY - tl.hy) * tl.hw + (AX - tl.hx)];
    double r = floor(__dadd_rn(v, 0.5));
    r = fmin(fmax(r, 0.0), 255.0);
    out[g] = static_cast<uint8_t>(r);
  }
}

}  // namespace

cudaError_t diffusion_launch(const uint8_t* img, const uint8_t* known, uint8_t* out, int W, int H,
                             const TileDesc* tiles, int n_tiles, const int64_t* foff,
                             const int64_t* poff, int64_t n_patches, int max_halo, int64_t max_core,
                             int iters, double* f0, double* f1, cudaStream_t s) {
  if (n_tiles == 0) return cudaSuccess;
  const unsigned gx = static_cast<unsigned>(std::min<int64_t>((max_halo + 255) / 256, 4096));
  diffusion_init_kernel<<<dim3(gx ? gx : 1, n_tiles), 256, 0, s>>>(img, known, W, H, tiles, n_tiles,
                                                                    foff, f0, f1);
  constexpr int S = 8;
  double* a = f0;
  double* b = f1;
  for (int done = 0; done < iters; done += S) {
    const int k = std::min(S, iters - done);
    diffusion_sweeps_kernel<S><<<static_cast<unsigned>(n_patches), 256, 0, s>>>(
        known, W, H, tiles, n_tiles, foff, poff, a, b, k);
    double* tmp = a;
    a = b;
    b = tmp;
  }
  const unsigned gc = static_cast<unsigned>(std::min<int64_t>((max_core + 255) / 256, 4096));
  diffusion_final_kernel<<<dim3(gc ? gc : 1, n_tiles), 256, 0, s>>>(known, out, W, H, tiles, n_tiles,
                                                                     foff, a);
  return cudaGetLastError();
}

}  // namespace tfb
