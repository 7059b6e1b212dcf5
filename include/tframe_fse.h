/*
 * tframe_fse.h — C-ABI of the B200-native FSE-lite hot path (libtframe_b200.so).
 *
 * Drop-in boundary for the reference's per-tile extrapolator and tiling
 * interface (tframe, arXiv 2207.00238 reference at /root/reference/proj):
 *
 *   reference interface (file:line)                       replaced by
 *   ----------------------------------------------------  ------------------------------
 *   tframe::plan_proposed(W,H,N)       tiling.hpp:99-111  tf_plan_proposed
 *   tframe::plan(Strategy::proposed..) tiling.hpp:301     tf_plan_proposed
 *   tframe::interior_boundary          tiling.hpp:231     tf_interior_boundary
 *   tframe::expand(tile,d,W,H)         overlap.hpp:25-34  tf_expand
 *   detail::check_fse_params           extrapolate.hpp:102 tf_check_fse_params
 *   registry_lookup("fse-lite",params) extrapolate.hpp:418 tf_fse_params_from_string
 *   FseLiteExtrapolator::params_string extrapolate.hpp:403 tf_fse_params_to_string
 *   FseLiteExtrapolator::influence_radius extrapolate.hpp:397 tf_influence_radius
 *   Extrapolator::extrapolate(img,mask) extrapolate.hpp:32 /
 *     fse_lite_extrapolate             extrapolate.hpp:263 tf_fse_extrapolate
 *   run_master / run_local             runtime.hpp:75,142 tf_tiled_extrapolate
 *   (blocks processed, FseLiteTrace::residual_energy.size()) tf_count_blocks
 *   diffusion_extrapolate              extrapolate.hpp:41-84 tf_diffusion_extrapolate
 *   run_master(algo "diffusion")       runtime.hpp:75       tf_tiled_diffusion
 *
 * Conventions: plain C, caller-owned buffers, no exceptions cross the
 * boundary.  Images are 8-bit row-major (stride = width, frames stacked);
 * masks are 8-bit, nonzero = known (image.hpp:53, PixelMask).  Every entry
 * point returns a tf_status; tf_last_error() gives the message of the last
 * failure on the calling thread.  Status codes mirror the reference's error
 * taxonomy / CLI exit codes (error.hpp:9-36, tools/main.cpp:18-22):
 * std::invalid_argument -> TF_EINVAL, TilingError -> TF_ETILING (exit code 4).
 *
 * There is no CPU fallback: compute entry points fail with TF_ECUDA when no
 * usable sm_100 device is present.
 */
#ifndef TFRAME_FSE_H
#define TFRAME_FSE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_ABI_VERSION 2

typedef enum tf_status {
  TF_OK = 0,
  TF_EINVAL = 1,       /* std::invalid_argument (params, dims)            */
  TF_EIO = 2,          /* reserved (IoError)                              */
  TF_EPROTO = 3,       /* reserved (ProtocolError / TransportError)       */
  TF_ETILING = 4,      /* TilingError: degenerate tiling                  */
  TF_ECUDA = 5,        /* CUDA runtime failure / no sm_100 device         */
  TF_ENCCL = 6,        /* NCCL failure                                    */
  TF_ENOMEM = 7,       /* host or device allocation failure               */
  TF_EUNSUPPORTED = 8  /* beyond the device path's index ranges (window
                          side > 2048, > 65535 blocks along a halo axis,
                          > 2^31 blocks a call)                           */
} tf_status;

/* Arithmetic mode of the FSE kernel. */
typedef enum tf_mode {
  TF_MODE_EXACT = 0, /* IEEE binary64, reference operation order, no FMA:
                        output byte-identical to the reference CPU FSE   */
  TF_MODE_FAST = 1   /* binary64 throughout (DFTs, W, update, 64-bit
                        argmax keys) with FMA contraction, on the Hermitian
                        half spectrum; blocks whose greedy selection meets
                        an argmax near-tie (2^-38 relative) or whose window
                        is nearly empty are re-run in EXACT arithmetic.
                        Within the north-star tolerance (>= 99.9 % of
                        reconstructed pixels within +-1, |dPSNR| <= 0.05 dB;
                        identical to EXACT on the c1-c5 frames measured) */
} tf_mode;

/* tiling.hpp:16-27 (Rect) */
typedef struct tf_rect {
  int32_t x, y, w, h;
} tf_rect;

/* extrapolate.hpp:86-92 (FseLiteParams): block_size, support_margin,
 * model_iterations, compensation (gamma), weight_decay (rho). */
typedef struct tf_fse_params {
  int32_t block;
  int32_t margin;
  int32_t iters;
  double gamma;
  double rho;
} tf_fse_params;

/* runtime.hpp:25-33 (RunStats) plus device-side counters. */
typedef struct tf_run_stats {
  int64_t plan_us;
  int64_t distribute_us;   /* H2D + launch issue                              */
  int64_t compute_span_us; /* dispatch end -> last GPU done                   */
  int64_t merge_us;        /* gather + D2H                                    */
  int64_t total_us;
  int64_t overhead_pixels; /* sum of halo minus core areas (overlap.hpp:21)  */
  int64_t blocks_reference;/* blocks the reference processes (all halo blocks
                              holding an unknown pixel, extrapolate.hpp:282) */
  int64_t blocks_processed;/* blocks the GPU ran: unknown pixel inside a core */
  double kernel_ms;        /* FSE kernel device time, max over GPUs           */
  double flops;            /* sum of F_b over processed blocks  */
  int64_t iterations;      /* sum of executed iterations I_b                  */
  int64_t pixels_evaluated;/* unknown core pixels written by the model        */
  double flops_executed;   /* FP64 flops the kernels actually execute (differs
                              from `flops` for the FAST half-spectrum kernel)  */
  int64_t blocks_refined;  /* FAST: blocks whose greedy selection met an argmax
                              near-tie and were re-run by the EXACT kernel     */
} tf_run_stats;

typedef struct tf_ctx tf_ctx;

/* ---- library / context ------------------------------------------------ */
int tf_abi_version(void);
/* n_gpus >= 1; device_ids may be NULL (devices 0..n_gpus-1).  Returns NULL on
 * failure (see tf_last_error(NULL)).  A context owns streams, device buffers
 * and pinned staging and serves one caller at a time: give each worker thread
 * its own (as each reference worker owns its Extrapolator, runtime.hpp) or
 * serialise calls on a shared one. */
tf_ctx* tf_create(int n_gpus, const int* device_ids);
void tf_destroy(tf_ctx* ctx);
const char* tf_last_error(const tf_ctx* ctx);
int tf_set_mode(tf_ctx* ctx, int mode);
int tf_get_mode(const tf_ctx* ctx);
int tf_device_count(int* out);

/* ---- parameters (registry semantics, extrapolate.hpp:342-437) ----------- */
int tf_check_fse_params(const tf_fse_params* p);
/* "block=..,margin=..,iters=..,gamma=..,rho=.." ; margin defaults to 2*block */
int tf_fse_params_from_string(const char* s, tf_fse_params* out);
int tf_fse_params_to_string(const tf_fse_params* p, char* buf, int buf_len);
int tf_influence_radius(const tf_fse_params* p);

/* ---- tiling (bit-exact with the reference) ------------------------------ */
int tf_plan_proposed(int W, int H, int N, tf_rect* out_tiles /* N */);
int tf_expand(const tf_rect* core, int d, int W, int H, tf_rect* out_halo);
long long tf_interior_boundary(const tf_rect* tiles, int n);
/* Blocks fse_lite_extrapolate processes on a w x h image (raster B-grid from
 * (0,0), blocks holding an unknown pixel); host-side, no GPU needed. */
int64_t tf_count_blocks(const uint8_t* known, int w, int h, int block);

/* ---- extrapolation ------------------------------------------------------- */
/* Extrapolator::extrapolate on one image: host buffers, synchronous. */
int tf_fse_extrapolate(tf_ctx* ctx, const uint8_t* img, const uint8_t* known, int w, int h,
                       const tf_fse_params* p, uint8_t* out);

/* run_master equivalent: plan -> expand -> FSE per halo -> crop -> merge, for
 * `frames` stacked W x H frames.  The (frame, tile) units are assigned to the
 * context's GPUs by LPT on core pixels (replaces the reference's i mod n,
 * runtime.hpp:102; equal costs give that round robin); every GPU receives only
 * the halo rectangles of its units (overlap.hpp:37-49), cores are gathered to
 * the first GPU over NCCL, then copied to `out`.  Output is independent of the
 * GPU count.  stats may be NULL. */
int tf_tiled_extrapolate(tf_ctx* ctx, const uint8_t* img, const uint8_t* known, int W, int H,
                         int frames, int tiles, int overlap, const tf_fse_params* p,
                         uint8_t* out, tf_run_stats* stats);

/* Device-resident variant on GPU `gpu` of the context: d_img/d_known/d_out
 * are device pointers on that GPU (d_out may alias nothing else); work is
 * enqueued on `stream` (a cudaStream_t, NULL = the context's stream) and NOT
 * synchronised.  A call made while `stream` is capturing a CUDA graph is
 * refused (TF_EINVAL); instead, the second of identical repeated calls is
 * captured by the library and later identical calls replay that graph.  Calls
 * on different streams are ordered by the library (each waits for the
 * previous call's kernels, which share per-GPU scratch).  Only the units that
 * tf_core_layout assigns to `part` of n_parts are computed (LPT on core pixels;
 * 0/1 = all); known pixels of the whole image are copied to d_out.  stats may
 * be NULL (filling it synchronises the stream). */
int tf_tiled_extrapolate_device(tf_ctx* ctx, int gpu, const uint8_t* d_img,
                                const uint8_t* d_known, int W, int H, int frames, int tiles,
                                int overlap, const tf_fse_params* p, int part, int n_parts,
                                uint8_t* d_out, void* stream, tf_run_stats* stats);

/* ---- diffusion extrapolator ---------------------------------
 * DiffusionExtrapolator::extrapolate / diffusion_extrapolate (extrapolate.hpp:41-84,
 * 367-386): K Jacobi sweeps of the 4-neighbour mean over the unknown pixels, byte-identical
 * to the reference.  iters < 1 -> TF_EINVAL ("diffusion_extrapolate: iterations must be >= 1"). */
int tf_diffusion_extrapolate(tf_ctx* ctx, const uint8_t* img, const uint8_t* known, int w, int h,
                             int iters, uint8_t* out);
/* run_master with algo "diffusion" (runtime.hpp:75-139): per-halo sweeps, cores merged. */
int tf_tiled_diffusion(tf_ctx* ctx, const uint8_t* img, const uint8_t* known, int W, int H,
                       int frames, int tiles, int overlap, int iters, uint8_t* out,
                       tf_run_stats* stats);

/* ---- image-quality metrics on the GPU (metrics.hpp:12-90) -----
 * Per frame of a frames x h x w batch (a = reference image, b = test image, known = mask,
 * nonzero = known, may be NULL).  mse / psnr / mse_missing are bit-identical to the
 * reference (integer sums, same final expressions); ssim's per-window values are
 * bit-identical and the mean over windows is summed in a fixed tree (deterministic, within
 * 1e-12 relative of the reference's sequential sum). */
typedef struct tf_quality_metrics {
  double mse;          /* mse(a, b) (metrics.hpp:12-24)                                  */
  double psnr;         /* psnr_from_mse(mse) (metrics.hpp:47-55); +inf when a == b         */
  double mse_missing;  /* over pixels with known == 0 (metrics.hpp:27-45); NaN if none      */
  double psnr_missing; /* psnr_from_mse(mse_missing); NaN if none                         */
  double ssim;         /* mean 8x8 SSIM (metrics.hpp:58-88); NaN if not asked or w|h < 8   */
  int64_t n_missing;   /* pixels with known == 0                                         */
} tf_quality_metrics;
/* Device buffers on GPU `gpu`, enqueued on `stream` (NULL: the context's stream); returns
 * after the results are on the host. */
int tf_quality_device(tf_ctx* ctx, int gpu, const uint8_t* d_a, const uint8_t* d_b,
                      const uint8_t* d_known, int w, int h, int frames, int want_ssim,
                      void* stream, tf_quality_metrics* out /* frames */);
/* Host buffers (copied to GPU 0 of the context). */
int tf_quality(tf_ctx* ctx, const uint8_t* a, const uint8_t* b, const uint8_t* known, int w,
               int h, int frames, int want_ssim, tf_quality_metrics* out /* frames */);
/* The reference's single-image functions on the GPU, same errors (std::invalid_argument ->
 * TF_EINVAL with the reference's message). */
int tf_mse(tf_ctx* ctx, const uint8_t* a, const uint8_t* b, int w, int h, double* out);
int tf_mse_missing(tf_ctx* ctx, const uint8_t* a, const uint8_t* b, const uint8_t* known, int w,
                   int h, double* out); /* no unknown pixel -> "mse_missing: mask has no unknown pixels" */
int tf_psnr(tf_ctx* ctx, const uint8_t* a, const uint8_t* b, int w, int h, double* out);
int tf_ssim(tf_ctx* ctx, const uint8_t* a, const uint8_t* b, int w, int h, double* out);
  /* w or h < 8 -> "ssim: image smaller than the 8x8 window" */
double tf_psnr_from_mse(double mse); /* metrics.hpp:47-50 */

/* ---- measurement ----------------------------------------------------------- */
/* Device durations (ms) of the most recent FSE kernel launches on GPU `gpu`
 * (oldest first, up to max_n; the context keeps the last 256).  Synchronises
 * the GPU's pending FSE launches.  Returns the count written, or -status. */
int tf_fse_kernel_times(tf_ctx* ctx, int gpu, float* out_ms, int max_n);
/* FP64 DFMA peak (TFLOP/s) and shared-memory LDS.128 bandwidth (TB/s) of a
 * device, measured with calibration kernels (roofline denominators). */
int tf_calibrate(int device, double* fp64_tflops, double* smem_tbs);
/* As tf_calibrate plus the FP64 tensor-core rate (mma.sync m8n8k4 .f64), the
 * FP64 datapath's measured maximum; any output may be NULL. */
int tf_calibrate_peaks(int device, double* dfma_tflops, double* dmma_tflops, double* smem_tbs);
/* Kernels this context has enqueued on GPU `gpu` so far (CUDA-graph replays
 * count their captured kernels). */
int tf_kernel_launches(tf_ctx* ctx, int gpu, int64_t* total);
/* Self-test: the FSE kernel's hoisted-reciprocal division must be bit-identical
 * to IEEE a/b; counts mismatches over n hashed operand pairs (expect 0). */
int tf_selftest_div(int device, int64_t n, uint64_t seed, int64_t* mismatches);

/* ---- multi-rank (one process per GPU, NCCL over NVLink) ------------------ */
/* 128-byte NCCL unique id, to be broadcast by the caller's bootstrap. */
int tf_comm_unique_id(uint8_t id[128]);
/* Attach an NCCL communicator to a single-GPU context. */
int tf_comm_init(tf_ctx* ctx, int nranks, int rank, const uint8_t id[128]);
/* Gather each rank's `bytes` at d_send into d_recv on `root` (rank-major,
 * nranks*bytes); non-root ranks may pass d_recv = NULL. */
int tf_comm_gather(tf_ctx* ctx, const void* d_send, void* d_recv, int64_t bytes, int root,
                   void* stream);
/* Host-side layout of the core gather (no GPU needed): for the frames*tiles
 * units (frame-major) gives each core rect, its frame, its owner part (LPT on
 * core pixels, ties by unit index, to the least-loaded part; replaces i mod n
 * of runtime.hpp:102) and its byte offset inside the owner's packed payload;
 * part_bytes[n_parts] receives each payload size. Any output may be NULL. */
int tf_core_layout(int W, int H, int frames, int tiles, int n_parts, tf_rect* cores,
                   int32_t* frame_of, int32_t* owner, int64_t* offs, int64_t* part_bytes);
/* Gather the cores of the units each rank owns (tf_core_layout with
 * n_parts = nranks) from every rank's frame-sized d_out into root's d_out
 * (same layout; run_master's collect + merge_into, runtime.hpp:112-130).
 * Packs, NCCL send/recv and unpacks on device, enqueued on `stream`. */
int tf_comm_gather_cores(tf_ctx* ctx, uint8_t* d_out, int W, int H, int frames, int tiles,
                         int root, void* stream);
/* One rank of a one-process-per-GPU job on HOST buffers (the run_master /
 * worker pair of runtime.hpp:60-139 for this rank): H2D of the halo
 * rectangles of the units this rank owns, FSE on them, NCCL gather of the
 * cores to `root`, D2H of the merged frames into `out` on root (other ranks
 * may pass out = NULL).  Without tf_comm_init it runs the whole job on the
 * context's GPU.  Synchronous.  io_bytes (may be NULL) receives {H2D bytes,
 * D2H bytes} of this rank. */
int tf_tiled_extrapolate_rank(tf_ctx* ctx, const uint8_t* img, const uint8_t* known, int W, int H,
                              int frames, int tiles, int overlap, const tf_fse_params* p, int root,
                              uint8_t* out, int64_t* io_bytes);

/* ---- synthetic inputs (versioned generator) ---------------- */
#define TF_SYNTH_VERSION 1
/* config in 1..5 (BASELINE configs); fills one W x H frame of image + mask
 * (mask 1 = known).  Seeds: image 1000*config + frame, mask that + 500. */
int tf_synth_frame(int config, int frame, int W, int H, uint8_t* img, uint8_t* known);

#ifdef __cplusplus
}
#endif

#endif /* TFRAME_FSE_H */
