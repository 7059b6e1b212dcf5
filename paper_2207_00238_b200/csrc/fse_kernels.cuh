// Device-side data layout shared by the host launcher and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tfb {

// One (frame, tile) unit: halo and core rects in absolute frame coordinates.
// The FSE block grid is anchored at the halo origin (extrapolate.hpp:278-279
// run on the extracted halo, runtime.hpp:98).
struct TileDesc {
  int32_t frame;
  int32_t hx, hy, hw, hh;  // halo (overlap.hpp:25-34)
  int32_t cx, cy, cw, ch;  // core
  int32_t gw, gh;          // block-grid dims: ceil(hw/B), ceil(hh/B)
  int32_t grid_off;        // prefix sum of gw*gh over previous tiles
  int32_t owner;           // part (GPU / rank) that reconstructs this unit (host LPT plan)
};

// One processed block: tile index + block-grid coordinates.
struct BlockDesc {
  uint32_t tile;
  uint16_t bxi, byi;
};

// Per-block counters (SURVEY §8(d) F_b terms), written by the FSE kernel.
struct BlockStat {
  int32_t M, L;      // support window = DFT size
  int32_t iters;     // executed iterations I_b
  int32_t pairs;     // non-self-conjugate selections P_b
  int32_t touched;   // touched bins T_b
  int32_t evaluated; // unknown core pixels evaluated (U_b restricted to the core)
};

struct FseLaunch {
  const uint8_t* img;
  const uint8_t* known;
  uint8_t* out;
  int32_t W, H;  // frame dims, row stride W, plane W*H
  const TileDesc* tiles;
  const BlockDesc* blocks;
  const int32_t* n_blocks;  // device counter written by the enumerator
  int32_t* next_block;      // work-queue head (zeroed before launch)
  int32_t B, margin, iters;
  double gamma;
  const double* rho_pow;  // rho^d, d = 0..margin (host std::pow, extrapolate.hpp:309)
  const double* tw;       // twiddles (cos,sin) interleaved, sizes n=1..wmax at n*(n-1)/2
  int32_t wmax;           // max window side in this launch
  BlockStat* stats;       // optional
  int32_t* wlog_kl;       // warp kernel: per-CTA selection log scratch (iters entries each)
  double2* wlog_c;
  unsigned char* scratch;  // big-window kernel: per-CTA spectra and model (BigLayout bytes each)
  int32_t nmax;            // big-window kernel: largest support window (bins) of the launch
  // FAST kernels: blocks whose greedy selection met an argmax near-tie are appended here
  // (and not evaluated); the EXACT kernel re-runs them afterwards (nullptr: no guard)
  BlockDesc* xlist;
  int32_t* n_xlist;
};

// Big-window kernel (windows past the shared-memory kernels' capacity, or selection logs too
// long for shared memory): per-CTA global scratch, 16-byte aligned sections
//   [W: N double2][R: N double2][row pass of w: N double2][of w*v: N double2]
//   [(w, w*v): N double2][first-touch positions: N int32][touched list: 2I int32]
//   [model values: 2I double2][selection log: I int32 + I double2]
struct BigLayout {
  size_t off_w, off_r, off_rw, off_rr, off_cw, off_post, off_lst, off_mval, off_logkl, off_logc, total;
  __host__ __device__ static size_t al(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }
  __host__ __device__ BigLayout(int nmax, int iters) {
    const size_t n = static_cast<size_t>(nmax), it = static_cast<size_t>(iters);
    off_w = 0;
    off_r = off_w + 16 * n;
    off_rw = off_r + 16 * n;
    off_rr = off_rw + 16 * n;
    off_cw = off_rr + 16 * n;
    off_post = off_cw + 16 * n;
    off_lst = al(off_post + 4 * n);
    off_mval = al(off_lst + 8 * it);
    off_logkl = off_mval + 32 * it;
    off_logc = al(off_logkl + 4 * it);
    total = al(off_logc + 16 * it);
  }
};
constexpr int kBigThreads = 512;

struct EnumLaunch {
  const uint8_t* known;
  int32_t W, H, B;
  const TileDesc* tiles;
  int32_t n_tiles;
  int32_t part, n_parts;      // only tiles with owner == part are enqueued
  BlockDesc* blocks;          // out: blocks for the CTA kernel
  int32_t* n_blocks;          // out: their count
  unsigned long long* ref_blocks;  // out, per tile: blocks the reference processes
  int32_t margin;
  int32_t warp_M, warp_L;     // windows of exactly this size go to the warp kernel (0 = none)
  BlockDesc* wblocks;         // out: blocks for the warp kernel
  int32_t* n_wblocks;
  // row band (streamed host path): only blocks whose first row, flattened over frames
  // (frame * H + halo y + block y), lies in [row0, row1) are counted and enqueued
  int64_t row0, row1;
  // FAST hybrid: a block whose support window has a known fraction below hyb_frac goes to
  // xblocks (run by the EXACT kernel: such windows are ill-conditioned)
  float hyb_frac;
  float hyb_ratio;            // ... or fewer known window pixels than hyb_ratio x the block's unknown ones
  BlockDesc* xblocks;
  int32_t* n_xblocks;
};
// device counters per launch slot: [n_blocks, next, n_wblocks, wnext, n_xblocks, xnext, -, -]
constexpr int kCounters = 8;

constexpr int kCY = 4;  // rows per DFT chunk
#ifndef TF_HALF_CY
#define TF_HALF_CY 4  // 8 measured slower (register spills)
#endif
constexpr int kHalfCY = TF_HALF_CY;  // rows per row-DFT chunk of the half kernels

// Shared-memory layout of the FSE kernel (bytes), computed identically on host and device.
//   [W replicated (2L x M or L x 2M double2, <= 2*nb)][twiddles: double2 x 2*wmax][union][slots][misc]
//   union = DFT phase {cwp, rw, rr: double2 x kCY*wmax; pix, kn: u8 x nb}
//         | loop phase {selection log: double2 x iters, int32 x iters}
//   after the loop the W region holds the model {mval: double2 x cap; lst: int32 x cap;
//   pos: int16 x nb} (cap = min(2I, nb) distinct touched bins).
#ifndef TF_CTA_HALF
#define TF_CTA_HALF 1  // FAST CTA kernel carries the Hermitian half spectrum (rows l <= L/2)
#endif
__host__ __device__ constexpr bool cta_half(bool exact) { return !exact && TF_CTA_HALF; }

struct SmemLayout {
  int nb, wmax, iters, nw, cap;
  int off_tw, off_union, off_pix, off_kn, off_lst, off_slots, off_misc, total;
  __host__ __device__ static int align16(int x) { return (x + 15) & ~15; }
  // nf = bins of the full window (W, window bytes, model); nb = bins the threads carry
  // (== nf except for the FAST half-spectrum CTA kernel)
  __host__ __device__ SmemLayout(int nb_, int wmax_, int iters_, int nw_, int nf = 0)
      : nb(nb_), wmax(wmax_), iters(iters_), nw(nw_) {
    if (nf < nb) nf = nb;
    cap = iters >= (nf + 1) / 2 ? nf : 2 * iters;
    off_tw = 32 * nf;
    off_union = off_tw + align16(2 * 16 * wmax);
    off_pix = off_union + 48 * kCY * wmax;
    off_kn = off_pix + nf;
    const int dft_end = off_kn + nf;
    off_lst = off_union + 16 * iters;  // int32 log after the double2 log
    const int loop_end = off_lst + 4 * iters;
    off_slots = align16(dft_end > loop_end ? dft_end : loop_end);
    off_misc = off_slots + 2 * nw * 32;
    total = off_misc + 16;
  }
};

// Warp-per-block kernel layout: [W replicated 2L x M: 32*N B][twiddles 32*wmax B][misc 16 B];
// the DFT scratch lives in W's second copy until the copy is written.
struct WarpLayout {
  int n, wmax, cap, off_tw, off_misc, off_log, total;
  __host__ __device__ WarpLayout(int n_, int wmax_, int iters) : n(n_), wmax(wmax_) {
    cap = iters >= (n + 1) / 2 ? n : 2 * iters;
    off_tw = 32 * n;
    off_misc = off_tw + 32 * wmax;
    total = off_misc + 16;
    off_log = (20 * cap + 2 * n + 15) & ~15;  // post-loop copy of the log inside W's space
  }
  __host__ __device__ bool fits(int n_, int wmax_, int iters) const {
    // DFT scratch in the second copy; post-loop model + log copy inside W's space
    return 48 * kCY * wmax_ + 2 * n_ <= 16 * n_ && off_log + 20 * iters <= 32 * n_;
  }
};

// FAST half-spectrum warp kernel layout: W rows 0..L-1 plus a copy of rows 0..lmax
// (the gathers touch rows 1..L+lmax only), the DFT scratch above row L until that copy
// is written; then the twiddles and misc.  lmax = bpth * (32 / M) - 1.
#ifndef TF_HALF_T2
#define TF_HALF_T2 1  // 32x32 half kernel: y-transform on the 17 half rows first, then x
#endif
constexpr int kHalfWB = 16;  // bytes per W element (binary64 complex)

// Windows up to 16 x 16 (one warp, <= 5 rows per lane) keep the selection log in shared
// memory (after the sync area) instead of a global scratch: short loops, where the per-
// iteration log store and the post-loop copy back were a visible share (config 3).
__host__ __device__ constexpr bool half_slog(int nt, int bpth, bool gen) {
  return !gen && nt == 32 && bpth <= 5;
}

#ifndef TF_HALF_NOCOPY
#define TF_HALF_NOCOPY 1  // full-window one-warp kernels: W without the copy of rows 0..lmax (c2 1.054 -> 0.990 ms)
#endif
__host__ __device__ constexpr bool half_nocopy(int nt, bool gen) { return TF_HALF_NOCOPY && nt == 32 && !gen; }

struct HalfLayout {
  int wbytes, off_tw, off_sync, off_log, total;
  // log_iters > 0: room for the selection log (double2 + int32 per iteration) at off_log.
  // nocopy: W keeps rows 0..L-1 plus the few rows (lmax - L/2 + 1) that the second gather
  // reaches past L-1; the first gather wraps by arithmetic instead of reading copy rows
  __host__ __device__ HalfLayout(int M, int L, int bpth, int wmax, int nt, int log_iters = 0,
                                 bool nocopy = false) {
    const int lmax = bpth * (nt / M) - 1;
    const int ncp = nocopy ? (lmax - L / 2 + 1 > 0 ? lmax - L / 2 + 1 : 0) : lmax + 1;
    const int rows = kHalfWB * M * (L + ncp);
    int scratch = 48 * kHalfCY * wmax + 2 * M * L;  // DFT scratch overlaps W (written after)
    if (nt == 32 && M == L && scratch < 32 * bpth * 32)
      scratch = 32 * bpth * 32;  // TF_HALF_T2: C(x, l) of the half rows, values + weights (FP64)
    wbytes = (rows > scratch ? rows : scratch);
    wbytes = (wbytes + 15) & ~15;
    off_tw = wbytes;
    off_sync = off_tw + 32 * wmax;  // twiddles x / y (FP64 complex)
    total = off_sync + 4 * 32 + 16;  // argmax slots (two warps), block id, sum of weights
    off_log = (total + 15) & ~15;
    if (log_iters > 0) total = off_log + 20 * log_iters;
  }
};

// FAST wide kernel (full windows S x S, 32 < S <= 64; fse_wide_kernel): NT threads, thread ->
// column k = tid mod S, row group tid / S (G = NT / S groups), rows l = group + G j <= S/2.
// wm: 0 = W stored FP32 complex (8 B), weights' DFT in FP32; 1 = weights' DFT in FP64, W
// stored FP32; 2 = FP64 throughout.
//   [region: W rows 0..S+HR+G-1 | DFT staging (w, w*v per pixel) | C(x, l) of the half rows |
//    post-loop selection log]
//   [twiddles: FP64 (cos, sin) x S, FP32 (cos, -sin) x S, FP32 (sin, cos) x S][slots][misc]
struct WideLayout {
  int nt, g, hr, bp, rows, region, off_tw, off_slots, off_misc, total;
  // S <= 48: three warps per block (two row groups, 12-13 bins per thread).  The per-
  // iteration argmax exchange costs every warp ~220 instructions whatever its share of the
  // bins, so fewer, fatter warps win: 192 / 160 / 96 / 64 threads -> c4 16.3 / 16.4 / 14.2 /
  // 15.7 ms, c5 (16 frames) 22.7 / 23.2 / 21.1 / 22.3 ms
#ifndef TF_WIDE_NT48
#define TF_WIDE_NT48 96
#endif
  __host__ __device__ static constexpr int threads(int S) { return S <= 48 ? TF_WIDE_NT48 : 256; }
  __host__ __device__ WideLayout(int S, int iters) {
    nt = threads(S);
    g = nt / S;
    hr = S / 2 + 1;
    bp = (hr + g - 1) / g;
    rows = S + hr + g;
    int r = 16 * S * rows;        // W (binary64 complex), copy rows included
    const int stage = 16 * S * S;  // w + w*v per window pixel
    const int cx = 32 * hr * S;    // C(x, l): values + weights
    const int lg = 20 * iters;     // selection log (double2 + int32 per iteration)
    r = r > stage ? r : stage;
    r = r > cx ? r : cx;
    r = r > lg ? r : lg;
    region = (r + 15) & ~15;
    off_tw = region;
    off_slots = off_tw + 16 * S;
    off_misc = off_slots + 2 * (nt / 32) * 32;
    total = off_misc + 16;
  }
};

// FAST pair kernel (full 16 x 16 windows, config 3): two blocks per warp, one per half-warp
// (lane -> column k, all 9 half-spectrum rows per lane).  Per half:
//   [region: W rows 0..S+HR-1 (binary64 complex) | first C(x, l) of the DFT] then, after both
//   halves, [selection logs: 2 x (double2 + int32) x iters][twiddles, rho^d][misc]
struct PairLayout {
  int region, off_log, log_stride, off_tw, total;
  // acc: the kernel's ACC variant accumulates the model at the core pixels in registers
  // (blocks of at most 16 pixels) and keeps no selection log
  __host__ __device__ PairLayout(int S, int iters, bool acc) {
    const int hr = S / 2 + 1;
    int r = 16 * S * (S + hr);                          // W rows 0..S-1 + copy of rows 0..hr-1 (FP64)
    const int stage = 16 * S * S, cx = 32 * hr * S;     // staging (w, w v); C(x, l) of both
    r = r > stage ? r : stage;
    r = r > cx ? r : cx;
    region = (r + 15) & ~15;
    off_log = 2 * region;
    log_stride = acc ? 0 : (20 * iters + 15) & ~15;  // per half: double2 x iters, then int32 x iters
    off_tw = off_log + 2 * log_stride;
    total = off_tw + 32 * S + 16;
  }
};

// ---- launch helpers (fse_kernels.cu)
struct KernelCfg {
  int nt, bpt;
};
constexpr int kNumCfgs = 10;
extern const KernelCfg kCfgs[kNumCfgs];
int pick_config(int nmax, bool exact);  // smallest config holding nmax bins, -1 if none
cudaError_t fse_prepare(int cfg, bool exact, int smem_bytes, int* ctas_per_sm);
cudaError_t fse_big_prepare(int* ctas_per_sm);
cudaError_t fse_big_launch(const FseLaunch& a, int grid, cudaStream_t s);
cudaError_t fse_launch(int cfg, bool exact, const FseLaunch& a, int grid, int smem_bytes,
                       cudaStream_t s);
// Diffusion extrapolator over the tiles' halos (diffusion.cu).  foff: FP64 field offset of
// each tile (prefix of hw*hh), poff: 32x32-patch offset of each tile; f0/f1: two fields of
// sum(hw*hh) doubles.  Writes the unknown core pixels of out.
cudaError_t diffusion_launch(const uint8_t* img, const uint8_t* known, uint8_t* out, int W, int H,
                             const TileDesc* tiles, int n_tiles, const int64_t* foff,
                             const int64_t* poff, int64_t n_patches, int max_halo, int64_t max_core,
                             int iters, double* f0, double* f1, cudaStream_t s);

// FFT twiddles (constant memory) from the size-32 cos/sin table: 32 x (cos, sin) of 2 pi j / 32
cudaError_t tw16_upload(const double* tw16);  // pair kernel's constant twiddles (16-point)
cudaError_t div_selftest_launch(long long n, unsigned long long seed, unsigned long long* bad,
                                cudaStream_t s);
// warp kernel variants: bins per lane (window M*L = 32*bpt with 32 % M == 0)
int pick_warp_bpt(int M, int L);  // 0 if no variant
cudaError_t fse_warp_prepare(int bpt, bool exact, int smem_bytes, int* ctas_per_sm);
cudaError_t fse_warp_launch(int bpt, bool exact, const FseLaunch& a, int grid, int smem_bytes,
                            cudaStream_t s);
// FAST-mode Hermitian half-spectrum warp kernel (window M = L in {8, 16, 32})
int pick_half_bpth(int nt, int M, int L);  // 0 if no variant
cudaError_t fse_half_prepare(int nt, int bpth, int smem_bytes, int* ctas_per_sm);
cudaError_t fse_half_launch(int nt, int bpth, const FseLaunch& a, int grid, int smem_bytes,
                                 cudaStream_t s);
// FAST wide kernel for full S x S windows, S in {40, 44, 48, 56, 64} (0 = no variant)
int wide_supported(int S);
cudaError_t fse_wide_prepare(int S, int smem_bytes, int* ctas_per_sm);
cudaError_t fse_wide_launch(int S, const FseLaunch& a, int grid, int smem_bytes, cudaStream_t s);
// Quality metrics (metrics.cu): per frame sse3[3f..3f+2] = {sum d^2, sum over unknown d^2,
// unknown count} (known may be null); with partial (ssim_partials doubles) and ssim_sum
// (frames doubles), the per-frame sum of the 8x8 window SSIM values.
int64_t ssim_partials(int w, int h, int frames);
cudaError_t quality_launch(const uint8_t* a, const uint8_t* b, const uint8_t* known, int w, int h,
                           int frames, int sms, unsigned long long* sse3, double* partial,
                           double* ssim_sum, cudaStream_t s);
// FAST pair kernel (S = 16 only; 0 if unsupported)
int pair_supported(int S);
cudaError_t fse_pair_prepare(int S, bool acc, int smem_bytes, int* warps_per_sm);
cudaError_t fse_pair_launch(int S, bool acc, const FseLaunch& a, int grid, int smem_bytes, cudaStream_t s);
cudaError_t enumerate_launch(const EnumLaunch& e, int max_grid_blocks, cudaStream_t s);
cudaError_t cores_launch(uint8_t* frames, int W, int H, const TileDesc* tiles, int n_tiles,
                         int part, int n_parts, const int64_t* offs, uint8_t* packed, bool unpack,
                         int64_t max_core, cudaStream_t s);

}  // namespace tfb
