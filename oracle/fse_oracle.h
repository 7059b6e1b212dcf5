/* TEST INFRASTRUCTURE ONLY — CPU oracle interface (see fse_oracle.c). */
#ifndef FSE_ORACLE_H
#define FSE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ETILING = 4, ORC_ENOMEM = 7 };

typedef struct {
  int32_t block, margin, iters;
  double gamma, rho;
} orc_params;

/* One record per processed block (raster order within an image). */
typedef struct {
  int32_t bx, by;     /* block origin, image-local */
  int32_t M, L;       /* support window (= DFT) size */
  int32_t iters;      /* executed iterations I_b */
  int32_t pairs;      /* non-self-conjugate selections P_b */
  int32_t touched;    /* touched bins T_b */
  int32_t unknown;    /* unknown pixels U_b */
  double min_gap;     /* min relative |R|^2 gap winner vs runner-up (divergence diagnostics) */
  int32_t gap_iter;   /* iteration of that minimum (-1: none) */
  int32_t pad;
} orc_block_stats;

int orc_plan_proposed(int W, int H, int N, int32_t* out_rects);
int orc_expand(const int32_t* core, int d, int W, int H, int32_t* halo);
int orc_check_params(const orc_params* p);
int orc_fse_lite(const uint8_t* img, const uint8_t* known, int w, int h, const orc_params* p,
                 uint8_t* out, orc_block_stats* stats, int64_t stats_cap, int64_t* n_blocks);
int orc_tiled(const uint8_t* img, const uint8_t* known, int W, int H, int frames, int tiles,
              int overlap, const orc_params* p, uint8_t* out, int64_t* blocks_per_tile);
/* diffusion extrapolator (extrapolate.hpp:41-84) and its tiled run (runtime.hpp:75-139) */
int orc_diffusion(const uint8_t* img, const uint8_t* known, int w, int h, int iters,
                  uint8_t* out);
int orc_tiled_diffusion(const uint8_t* img, const uint8_t* known, int W, int H, int frames,
                        int tiles, int overlap, int iters, uint8_t* out);

/* metrics.hpp:12-88 */
double orc_mse(const uint8_t* a, const uint8_t* b, int w, int h);
int orc_mse_missing(const uint8_t* a, const uint8_t* b, const uint8_t* known, int w, int h,
                    double* out);
double orc_psnr_from_mse(double m);
double orc_ssim(const uint8_t* a, const uint8_t* b, int w, int h);

#ifdef __cplusplus
}
#endif
#endif
