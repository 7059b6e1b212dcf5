/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the FSE-lite hot path.
 *
 * Plain-C restatement of the reference algorithm (tframe, /root/reference/proj)
 * used as the CHECKER by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  The product library never links or calls it.
 *
 * Parity pin: the restatement is checked bit-for-bit against the compiled,
 * unmodified reference (oracle/_ref/libtframe_ref.so, built by oracle/Makefile)
 * and against the golden fixtures in tests/golden/ that the reference itself
 * produced (tests/golden/make_golden.py).  See tests/test_oracle.py.
 *
 * Floating-point contract: every operation below is one IEEE-754 binary64
 * operation with round-to-nearest and NO contraction (build with
 * -ffp-contract=off), in the same order as the reference compiled by g++ for
 * x86-64 (no FMA): std::complex<double> products are (ac - bd, ad + bc),
 * real*complex and complex/real are component-wise, std::norm is x*x + y*y.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "fse_oracle.h"

/* ---------------------------------------------------------------- tiling */

static int cmp_rect_yx(const void* a, const void* b) {
  const int32_t* ra = (const int32_t*)a;
  const int32_t* rb = (const int32_t*)b;
  if (ra[1] != rb[1]) return ra[1] < rb[1] ? -1 : 1;
  if (ra[0] != rb[0]) return ra[0] < rb[0] ? -1 : 1;
  return 0;
}

/* tiling.hpp:60-92 (plan_proposed_landscape); rects are {x, y, w, h}. */
static int plan_landscape(int W, int H, int N, int32_t* out) {
  const double r = (double)W / (double)H;
  long long nr = llround(sqrt((double)N / r));
  const int n_rows = nr < 1 ? 1 : (int)nr;
  int y = 0, t = 0;
  for (int i = 1; i <= n_rows; ++i) {
    const int n_cols = (i <= N % n_rows) ? (N + n_rows - 1) / n_rows : N / n_rows;
    if (n_cols < 1) return ORC_ETILING;
    long long h = (long long)H * n_cols / N + ((long long)H * n_cols % N) / n_rows;
    if (i == n_rows) h = H - y;
    if (h < 1) return ORC_ETILING;
    int x = 0;
    for (int j = 1; j <= n_cols; ++j) {
      const int w = (j <= W % n_cols) ? W / n_cols + 1 : W / n_cols;
      if (w < 1) return ORC_ETILING;
      out[4 * t + 0] = x;
      out[4 * t + 1] = y;
      out[4 * t + 2] = w;
      out[4 * t + 3] = (int)h;
      ++t;
      x += w;
    }
    y += (int)h;
  }
  if (y != H) return ORC_ETILING;
  return t == N ? ORC_OK : ORC_ETILING;
}

/* tiling.hpp:99-111 (plan_proposed). */
int orc_plan_proposed(int W, int H, int N, int32_t* out) {
  if (W < 1 || H < 1 || N < 1) return ORC_EINVAL;
  if ((long long)N > (long long)W * H) return ORC_ETILING;
  if (W >= H) return plan_landscape(W, H, N, out);
  int rc = plan_landscape(H, W, N, out);
  if (rc != ORC_OK) return rc;
  for (int i = 0; i < N; ++i) {
    int32_t x = out[4 * i], y = out[4 * i + 1], w = out[4 * i + 2], h = out[4 * i + 3];
    out[4 * i] = y;
    out[4 * i + 1] = x;
    out[4 * i + 2] = h;
    out[4 * i + 3] = w;
  }
  qsort(out, (size_t)N, 4 * sizeof(int32_t), cmp_rect_yx);
  return ORC_OK;
}

/* overlap.hpp:25-34 (expand). */
int orc_expand(const int32_t* core, int d, int W, int H, int32_t* halo) {
  if (d < 0) return ORC_EINVAL;
  if (core[0] < 0 || core[1] < 0 || core[0] + core[2] > W || core[1] + core[3] > H)
    return ORC_EINVAL;
  const int x0 = core[0] - d > 0 ? core[0] - d : 0;
  const int y0 = core[1] - d > 0 ? core[1] - d : 0;
  const int x1 = core[0] + core[2] + d < W ? core[0] + core[2] + d : W;
  const int y1 = core[1] + core[3] + d < H ? core[1] + core[3] + d : H;
  halo[0] = x0;
  halo[1] = y0;
  halo[2] = x1 - x0;
  halo[3] = y1 - y0;
  return ORC_OK;
}

/* extrapolate.hpp:102-110 (check_fse_params). */
int orc_check_params(const orc_params* p) {
  if (p->block < 2) return ORC_EINVAL;
  if (p->margin < 0) return ORC_EINVAL;
  if (p->iters < 1) return ORC_EINVAL;
  if (p->gamma <= 0.0 || p->gamma > 1.0) return ORC_EINVAL;
  if (p->rho <= 0.0 || p->rho >= 1.0) return ORC_EINVAL;
  return ORC_OK;
}

/* ------------------------------------------------------------ FSE-lite */

typedef struct {
  int M, L, N;
  double *twx_c, *twx_s, *twy_c, *twy_s; /* extrapolate.hpp:200-207 */
  double *W_re, *W_im, *R_re, *R_im, *rows_re, *rows_im, *weighted;
  double *mod_re, *mod_im; /* model_, indexed by bin */
  uint8_t* touched;
  int* list;
  int n_list;
} model_t;

static void make_twiddles(int m, double* c, double* s) {
  for (int i = 0; i < m; ++i) {
    const double a = 2.0 * M_PI * i / m;
    c[i] = cos(a);
    s[i] = sin(a);
  }
}

static int model_init(model_t* md, int M, int L) {
  memset(md, 0, sizeof(*md));
  md->M = M;
  md->L = L;
  md->N = M * L;
  const size_t n = (size_t)md->N;
  md->twx_c = malloc(sizeof(double) * (size_t)M);
  md->twx_s = malloc(sizeof(double) * (size_t)M);
  md->twy_c = malloc(sizeof(double) * (size_t)L);
  md->twy_s = malloc(sizeof(double) * (size_t)L);
  double* big = malloc(sizeof(double) * n * 9);
  md->touched = malloc(n);
  md->list = malloc(sizeof(int) * n);
  if (!md->twx_c || !md->twx_s || !md->twy_c || !md->twy_s || !big || !md->touched || !md->list)
    return ORC_ENOMEM;
  md->W_re = big;
  md->W_im = big + n;
  md->R_re = big + 2 * n;
  md->R_im = big + 3 * n;
  md->rows_re = big + 4 * n;
  md->rows_im = big + 5 * n;
  md->weighted = big + 6 * n;
  md->mod_re = big + 7 * n;
  md->mod_im = big + 8 * n;
  make_twiddles(M, md->twx_c, md->twx_s);
  make_twiddles(L, md->twy_c, md->twy_s);
  return ORC_OK;
}

static void model_free(model_t* md) {
  free(md->twx_c);
  free(md->twx_s);
  free(md->twy_c);
  free(md->twy_s);
  free(md->W_re);
  free(md->touched);
  free(md->list);
}

/* extrapolate.hpp:210-228 (dft2): out(k,l) = sum in(x,y) e^{-j2pi(kx/M+ly/L)},
 * row pass over x (real * conj(tw)), then column pass over y (complex *
 * conj(tw)); output index l*M + k. */
static void dft2(model_t* md, const double* in, double* out_re, double* out_im) {
  const int M = md->M, L = md->L;
  for (int y = 0; y < L; ++y)
    for (int k = 0; k < M; ++k) {
      double ar = 0.0, ai = 0.0;
      for (int x = 0; x < M; ++x) {
        const int t = (k * x) % M;
        const double v = in[y * M + x];
        ar += v * md->twx_c[t];
        ai += v * -md->twx_s[t];
      }
      md->rows_re[y * M + k] = ar;
      md->rows_im[y * M + k] = ai;
    }
  for (int k = 0; k < M; ++k)
    for (int l = 0; l < L; ++l) {
      double ar = 0.0, ai = 0.0;
      for (int y = 0; y < L; ++y) {
        const int t = (l * y) % L;
        const double a = md->rows_re[y * M + k], b = md->rows_im[y * M + k];
        const double c = md->twy_c[t], d = -md->twy_s[t];
        ar += a * c - b * d;
        ai += a * d + b * c;
      }
      out_re[l * M + k] = ar;
      out_im[l * M + k] = ai;
    }
}

static void add_to_model(model_t* md, int u, int v, double cr, double ci) {
  const int i = v * md->M + u;
  md->mod_re[i] += cr;
  md->mod_im[i] += ci;
  if (!md->touched[i]) {
    md->touched[i] = 1;
    md->list[md->n_list++] = i;
  }
}

/* extrapolate.hpp:126-186 (FseWindowModel::fit), energy trace omitted. */
static void fit(model_t* md, const double* weights, const double* values, const orc_params* p,
                orc_block_stats* st) {
  const int M = md->M, L = md->L, N = md->N;
  md->n_list = 0;
  for (int i = 0; i < N; ++i) {
    md->mod_re[i] = 0.0;
    md->mod_im[i] = 0.0;
    md->touched[i] = 0;
  }
  dft2(md, weights, md->W_re, md->W_im);
  for (int i = 0; i < N; ++i) md->weighted[i] = weights[i] * values[i];
  dft2(md, md->weighted, md->R_re, md->R_im);
  const double wsum = md->W_re[0];
  if (st) {
    st->iters = 0;
    st->pairs = 0;
    st->min_gap = INFINITY;
    st->gap_iter = -1;
  }
  if (wsum <= 0.0) return;
  for (int it = 0; it < p->iters; ++it) {
    int best = 0;
    double best_mag = 0.0, second = 0.0;
    for (int i = 0; i < N; ++i) {
      const double m = md->R_re[i] * md->R_re[i] + md->R_im[i] * md->R_im[i];
      if (m > best_mag) {
        best_mag = m;
        best = i;
      }
    }
    if (best_mag == 0.0) break;
    const int u = best % M, v = best / M;
    const int u2 = (M - u) % M, v2 = (L - v) % L;
    const int self_conj = (u2 == u && v2 == v);
    if (st) {
      /* divergence diagnostics: relative gap between the winner and the best
       * bin that is neither the winner nor its conjugate partner */
      const int partner = v2 * M + u2;
      for (int i = 0; i < N; ++i) {
        if (i == best || i == partner) continue;
        const double m = md->R_re[i] * md->R_re[i] + md->R_im[i] * md->R_im[i];
        if (m > second) second = m;
      }
      const double gap = (best_mag - second) / best_mag;
      if (gap < st->min_gap) {
        st->min_gap = gap;
        st->gap_iter = it;
      }
    }
    const double cr = (p->gamma * md->R_re[best]) / wsum;
    const double ci = (p->gamma * md->R_im[best]) / wsum;
    add_to_model(md, u, v, cr, ci);
    if (!self_conj) add_to_model(md, u2, v2, cr, -ci);
    for (int l = 0; l < L; ++l) {
      int l1 = (l - v) % L;
      if (l1 < 0) l1 += L;
      int l2 = (l - v2) % L;
      if (l2 < 0) l2 += L;
      for (int k = 0; k < M; ++k) {
        const int i = l * M + k;
        int k1 = (k - u) % M;
        if (k1 < 0) k1 += M;
        const double c = md->W_re[l1 * M + k1], d = md->W_im[l1 * M + k1];
        md->R_re[i] -= cr * c - ci * d;
        md->R_im[i] -= cr * d + ci * c;
        if (!self_conj) {
          int k2 = (k - u2) % M;
          if (k2 < 0) k2 += M;
          const double c2 = md->W_re[l2 * M + k2], d2 = md->W_im[l2 * M + k2];
          const double nci = -ci;
          md->R_re[i] -= cr * c2 - nci * d2;
          md->R_im[i] -= cr * d2 + nci * c2;
        }
      }
    }
    if (st) {
      st->iters += 1;
      st->pairs += self_conj ? 0 : 1;
    }
  }
  if (st) st->touched = md->n_list;
}

/* extrapolate.hpp:189-197 (evaluate). */
static double evaluate(const model_t* md, int x, int y) {
  double acc = 0.0;
  for (int j = 0; j < md->n_list; ++j) {
    const int i = md->list[j];
    const int k = i % md->M, l = i / md->M;
    const int tx = (k * x) % md->M, ty = (l * y) % md->L;
    const double mr = md->mod_re[i], mi = md->mod_im[i];
    const double cx = md->twx_c[tx], sx = md->twx_s[tx];
    const double cy = md->twy_c[ty], sy = md->twy_s[ty];
    const double tr = mr * cx - mi * sx;
    const double ti = mr * sx + mi * cx;
    acc += tr * cy - ti * sy;
  }
  return acc;
}

typedef struct {
  int M, L;
  model_t md;
} cache_entry;

/* extrapolate.hpp:263-340 (fse_lite_extrapolate).  stats (optional) receives
 * one record per processed block, in raster order; *n_blocks its count. */
int orc_fse_lite(const uint8_t* img, const uint8_t* known, int w, int h, const orc_params* p,
                 uint8_t* out, orc_block_stats* stats, int64_t stats_cap, int64_t* n_blocks) {
  if (w < 1 || h < 1) return ORC_EINVAL;
  int rc = orc_check_params(p);
  if (rc != ORC_OK) return rc;
  const int B = p->block, margin = p->margin;
  memcpy(out, img, (size_t)w * h);
  cache_entry* cache = NULL;
  int n_cache = 0;
  int64_t nb = 0;
  const int maxM = (B + 2 * margin) < w ? (B + 2 * margin) : w;
  const int maxL = (B + 2 * margin) < h ? (B + 2 * margin) : h;
  double* weights = malloc(sizeof(double) * (size_t)maxM * maxL);
  double* values = malloc(sizeof(double) * (size_t)maxM * maxL);
  double* rho_pow = malloc(sizeof(double) * (size_t)(margin + 1));
  if (!weights || !values || !rho_pow) return ORC_ENOMEM;
  for (int dd = 0; dd <= margin; ++dd) rho_pow[dd] = pow(p->rho, (double)dd);

  for (int by = 0; by < h; by += B)
    for (int bx = 0; bx < w; bx += B) {
      const int bw = B < w - bx ? B : w - bx;
      const int bh = B < h - by ? B : h - by;
      int has_unknown = 0;
      for (int y = by; y < by + bh && !has_unknown; ++y)
        for (int x = bx; x < bx + bw; ++x)
          if (!known[(size_t)y * w + x]) {
            has_unknown = 1;
            break;
          }
      if (!has_unknown) continue;
      const int sx0 = bx - margin > 0 ? bx - margin : 0;
      const int sy0 = by - margin > 0 ? by - margin : 0;
      const int sx1 = bx + bw + margin < w ? bx + bw + margin : w;
      const int sy1 = by + bh + margin < h ? by + bh + margin : h;
      const int sw = sx1 - sx0, sh = sy1 - sy0;

      model_t* md = NULL;
      for (int c = 0; c < n_cache; ++c)
        if (cache[c].M == sw && cache[c].L == sh) md = &cache[c].md;
      if (!md) {
        cache = realloc(cache, sizeof(cache_entry) * (size_t)(n_cache + 1));
        cache[n_cache].M = sw;
        cache[n_cache].L = sh;
        rc = model_init(&cache[n_cache].md, sw, sh);
        if (rc != ORC_OK) return rc;
        md = &cache[n_cache].md;
        ++n_cache;
      }
      int any_known = 0;
      for (int y = sy0; y < sy1; ++y)
        for (int x = sx0; x < sx1; ++x) {
          const int i = (y - sy0) * sw + (x - sx0);
          weights[i] = 0.0;
          values[i] = 0.0;
          if (!known[(size_t)y * w + x]) continue;
          any_known = 1;
          int dx = bx - x, t = x - (bx + bw - 1);
          if (t > dx) dx = t;
          if (dx < 0) dx = 0;
          int dy = by - y;
          t = y - (by + bh - 1);
          if (t > dy) dy = t;
          if (dy < 0) dy = 0;
          weights[i] = rho_pow[dx > dy ? dx : dy];
          values[i] = (double)img[(size_t)y * w + x];
        }
      orc_block_stats* st = (stats && nb < stats_cap) ? &stats[nb] : NULL;
      if (st) {
        st->bx = bx;
        st->by = by;
        st->M = sw;
        st->L = sh;
        st->unknown = 0;
      }
      fit(md, weights, values, p, st);
      for (int y = by; y < by + bh; ++y)
        for (int x = bx; x < bx + bw; ++x) {
          if (known[(size_t)y * w + x]) continue;
          if (st) st->unknown += 1;
          if (!any_known) {
            out[(size_t)y * w + x] = 128;
            continue;
          }
          double v = floor(evaluate(md, x - sx0, y - sy0) + 0.5);
          if (v < 0.0) v = 0.0;
          if (v > 255.0) v = 255.0;
          out[(size_t)y * w + x] = (uint8_t)v;
        }
      ++nb;
    }
  for (int c = 0; c < n_cache; ++c) model_free(&cache[c].md);
  free(cache);
  free(weights);
  free(values);
  free(rho_pow);
  if (n_blocks) *n_blocks = nb;
  return ORC_OK;
}

/* runtime.hpp:75-139 (run_master) semantics, sequential: plan, expand, run
 * FSE-lite on every halo (frames stacked), crop the core, merge. */
int orc_tiled(const uint8_t* img, const uint8_t* known, int W, int H, int frames, int tiles,
              int overlap, const orc_params* p, uint8_t* out, int64_t* blocks_per_tile) {
  int32_t* rects = malloc(sizeof(int32_t) * 4 * (size_t)tiles);
  if (!rects) return ORC_ENOMEM;
  int rc = orc_plan_proposed(W, H, tiles, rects);
  if (rc != ORC_OK) {
    free(rects);
    return rc;
  }
  for (int f = 0; f < frames; ++f) {
    const size_t plane = (size_t)W * H * f;
    for (int t = 0; t < tiles; ++t) {
      int32_t halo[4];
      rc = orc_expand(&rects[4 * t], overlap, W, H, halo);
      if (rc != ORC_OK) break;
      const size_t hn = (size_t)halo[2] * halo[3];
      uint8_t* si = malloc(hn);
      uint8_t* sm = malloc(hn);
      uint8_t* so = malloc(hn);
      for (int y = 0; y < halo[3]; ++y) {
        memcpy(si + (size_t)y * halo[2], img + plane + (size_t)(halo[1] + y) * W + halo[0],
               (size_t)halo[2]);
        memcpy(sm + (size_t)y * halo[2], known + plane + (size_t)(halo[1] + y) * W + halo[0],
               (size_t)halo[2]);
      }
      int64_t nb = 0;
      rc = orc_fse_lite(si, sm, halo[2], halo[3], p, so, NULL, 0, &nb);
      if (rc == ORC_OK) {
        if (blocks_per_tile) blocks_per_tile[(size_t)f * tiles + t] = nb;
        const int ox = rects[4 * t] - halo[0], oy = rects[4 * t + 1] - halo[1];
        for (int y = 0; y < rects[4 * t + 3]; ++y)
          memcpy(out + plane + (size_t)(rects[4 * t + 1] + y) * W + rects[4 * t],
                 so + (size_t)(oy + y) * halo[2] + ox, (size_t)rects[4 * t + 2]);
      }
      free(si);
      free(sm);
      free(so);
      if (rc != ORC_OK) break;
    }
    if (rc != ORC_OK) break;
  }
  free(rects);
  return rc;
}

/* ---- diffusion extrapolator (extrapolate.hpp:41-84): K Jacobi sweeps, unknown pixels start
 * at 128 and take the mean of their in-bounds 4-neighbours (left, right, up, down summed in
 * that order, then divided by the count); known pixels fixed; floor(v + 0.5) clamped. */
int orc_diffusion(const uint8_t* img, const uint8_t* known, int w, int h, int iters,
                  uint8_t* out) {
  if (w < 1 || h < 1) return ORC_EINVAL;
  if (iters < 1) return ORC_EINVAL;
  const size_t n = (size_t)w * h;
  double* cur = malloc(sizeof(double) * n);
  double* nxt = malloc(sizeof(double) * n);
  if (!cur || !nxt) {
    free(cur);
    free(nxt);
    return ORC_ENOMEM;
  }
  for (size_t i = 0; i < n; ++i) cur[i] = known[i] ? (double)img[i] : 128.0;
  memcpy(nxt, cur, sizeof(double) * n);
  for (int it = 0; it < iters; ++it) {
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const size_t i = (size_t)y * w + x;
        if (known[i]) continue;
        double sum = 0.0;
        int cnt = 0;
        if (x > 0) { sum += cur[i - 1]; ++cnt; }
        if (x + 1 < w) { sum += cur[i + 1]; ++cnt; }
        if (y > 0) { sum += cur[i - (size_t)w]; ++cnt; }
        if (y + 1 < h) { sum += cur[i + (size_t)w]; ++cnt; }
        nxt[i] = cnt > 0 ? sum / cnt : 128.0;
      }
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  for (size_t i = 0; i < n; ++i) {
    if (known[i]) {
      out[i] = img[i];
    } else {
      double v = floor(cur[i] + 0.5);
      v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
      out[i] = (uint8_t)v;
    }
  }
  free(cur);
  free(nxt);
  return ORC_OK;
}

/* run_master with the diffusion extrapolator per halo (runtime.hpp:75-139). */
int orc_tiled_diffusion(const uint8_t* img, const uint8_t* known, int W, int H, int frames,
                        int tiles, int overlap, int iters, uint8_t* out) {
  int32_t* rects = malloc(sizeof(int32_t) * 4 * (size_t)tiles);
  if (!rects) return ORC_ENOMEM;
  int rc = orc_plan_proposed(W, H, tiles, rects);
  for (int f = 0; rc == ORC_OK && f < frames; ++f) {
    const size_t plane = (size_t)W * H * f;
    for (int t = 0; rc == ORC_OK && t < tiles; ++t) {
      int32_t halo[4];
      rc = orc_expand(&rects[4 * t], overlap, W, H, halo);
      if (rc != ORC_OK) break;
      const size_t hn = (size_t)halo[2] * halo[3];
      uint8_t* si = malloc(hn);
      uint8_t* sm = malloc(hn);
      uint8_t* so = malloc(hn);
      for (int y = 0; y < halo[3]; ++y) {
        memcpy(si + (size_t)y * halo[2], img + plane + (size_t)(halo[1] + y) * W + halo[0],
               (size_t)halo[2]);
        memcpy(sm + (size_t)y * halo[2], known + plane + (size_t)(halo[1] + y) * W + halo[0],
               (size_t)halo[2]);
      }
      rc = orc_diffusion(si, sm, halo[2], halo[3], iters, so);
      if (rc == ORC_OK) {
        const int ox = rects[4 * t] - halo[0], oy = rects[4 * t + 1] - halo[1];
        for (int y = 0; y < rects[4 * t + 3]; ++y)
          memcpy(out + plane + (size_t)(rects[4 * t + 1] + y) * W + rects[4 * t],
                 so + (size_t)(oy + y) * halo[2] + ox, (size_t)rects[4 * t + 2]);
      }
      free(si);
      free(sm);
      free(so);
    }
  }
  free(rects);
  return rc;
}

/* ---------------------------------------------------------------- metrics
 * metrics.hpp:12-88 restated: binary64 accumulation in raster order, the same
 * expressions (the checker for the GPU quality kernels). */

double orc_mse(const uint8_t* a, const uint8_t* b, int w, int h) {
  /* metrics.hpp:12-24 */
  double sum = 0.0;
  const size_t n = (size_t)w * h;
  for (size_t i = 0; i < n; ++i) {
    const double d = (double)a[i] - (double)b[i];
    sum += d * d;
  }
  return sum / (double)n;
}

int orc_mse_missing(const uint8_t* a, const uint8_t* b, const uint8_t* known, int w, int h,
                    double* out) {
  /* metrics.hpp:27-45: pixels the mask marks unknown; none -> error */
  double sum = 0.0;
  size_t n = 0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      if (known[i]) continue;
      const double d = (double)a[i] - (double)b[i];
      sum += d * d;
      ++n;
    }
  if (n == 0) return ORC_EINVAL;
  *out = sum / (double)n;
  return ORC_OK;
}

double orc_psnr_from_mse(double m) {
  /* metrics.hpp:47-50 */
  if (m == 0.0) return INFINITY;
  return 10.0 * log10(255.0 * 255.0 / m);
}

double orc_ssim(const uint8_t* a, const uint8_t* b, int w, int h) {
  /* metrics.hpp:58-88: uniform 8x8 windows, stride 1; NaN when smaller than 8x8 */
  if (w < 8 || h < 8) return NAN;
  const double c1 = (0.01 * 255.0) * (0.01 * 255.0);
  const double c2 = (0.03 * 255.0) * (0.03 * 255.0);
  const double inv_n = 1.0 / (8 * 8);
  double total = 0.0;
  size_t windows = 0;
  for (int wy = 0; wy + 8 <= h; ++wy)
    for (int wx = 0; wx + 8 <= w; ++wx) {
      double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
      for (int y = wy; y < wy + 8; ++y)
        for (int x = wx; x < wx + 8; ++x) {
          const double va = a[(size_t)y * w + x];
          const double vb = b[(size_t)y * w + x];
          sa += va;
          sb += vb;
          saa += va * va;
          sbb += vb * vb;
          sab += va * vb;
        }
      const double mu_a = sa * inv_n;
      const double mu_b = sb * inv_n;
      const double var_a = saa * inv_n - mu_a * mu_a;
      const double var_b = sbb * inv_n - mu_b * mu_b;
      const double cov = sab * inv_n - mu_a * mu_b;
      total += ((2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2)) /
               ((mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2));
      ++windows;
    }
  return total / (double)windows;
}
