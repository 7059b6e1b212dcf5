// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C shim over the UNMODIFIED reference headers (tframe, header-only C++20),
// compiled from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/libtframe_ref.so.  It is the ground truth the C restatement
// (oracle/fse_oracle.c) and the CUDA path are checked against, and the
// "reference" CPU arm of bench.py.  No reference source is copied here: this
// file only calls the reference's public functions.
//
//   ref_plan_proposed   -> tframe::plan_proposed          (tiling.hpp:99)
//   ref_expand          -> tframe::expand                 (overlap.hpp:25)
//   ref_fse_lite        -> tframe::fse_lite_extrapolate   (extrapolate.hpp:263)
//   ref_registry        -> tframe::registry_lookup        (extrapolate.hpp:418)
//   ref_run_local       -> tframe::run_local              (runtime.hpp:142)
//   ref_tiled_allcores  -> bit-exact band split of fse_lite_extrapolate on a
//                          thread pool (SURVEY §8(d) "all host cores")
//   ref_gen_scatter_mask, ref_make_scene, ref_psnr, ref_ssim -> pgm/bench/metrics
//   ref_synth_frame     -> the repo's versioned input generator (synth_gen.hpp, header-only,
//                          the same source as the product's tf_synth_frame), so bench.py's
//                          reference arm builds its inputs without the product library

#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "tframe/tframe.hpp"
#include "synth_gen.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

tframe::ImageBuffer to_image(const uint8_t* p, int w, int h) {
  return tframe::ImageBuffer(w, h, std::vector<uint8_t>(p, p + static_cast<size_t>(w) * h));
}

tframe::PixelMask to_mask(const uint8_t* p, int w, int h) {
  tframe::PixelMask m(w, h);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) m.set_known(x, y, p[static_cast<size_t>(y) * w + x] != 0);
  return m;
}

std::string params_str(int block, int margin, int iters, double gamma, double rho) {
  tframe::FseLiteParams p;
  p.block_size = block;
  p.support_margin = margin;
  p.model_iterations = iters;
  p.compensation = gamma;
  p.weight_decay = rho;
  return tframe::FseLiteExtrapolator(p).params_string();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_plan_proposed(int W, int H, int N, int32_t* out /* 4*N */) {
  try {
    const tframe::TileLayout t = tframe::plan_proposed(W, H, N);
    for (size_t i = 0; i < t.tiles.size(); ++i) {
      out[4 * i + 0] = t.tiles[i].x;
      out[4 * i + 1] = t.tiles[i].y;
      out[4 * i + 2] = t.tiles[i].w;
      out[4 * i + 3] = t.tiles[i].h;
    }
    return 0;
  } catch (const tframe::TilingError& e) {
    return fail(e, 4);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

long long ref_interior_boundary(int W, int H, int N) {
  return tframe::interior_boundary(tframe::plan_proposed(W, H, N));
}

int ref_expand(const int32_t* core, int d, int W, int H, int32_t* halo) {
  try {
    const auto et = tframe::expand(tframe::Rect{core[0], core[1], core[2], core[3]}, d, W, H);
    halo[0] = et.halo.x;
    halo[1] = et.halo.y;
    halo[2] = et.halo.w;
    halo[3] = et.halo.h;
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  }
}

// n_blocks (optional): number of blocks the reference processes (== size of
// FseLiteTrace::residual_energy, extrapolate.hpp:313-317).
int ref_fse_lite(const uint8_t* img, const uint8_t* known, int w, int h, int block, int margin,
                 int iters, double gamma, double rho, uint8_t* out, int64_t* n_blocks) {
  try {
    tframe::FseLiteParams p;
    p.block_size = block;
    p.support_margin = margin;
    p.model_iterations = iters;
    p.compensation = gamma;
    p.weight_decay = rho;
    tframe::FseLiteTrace trace;
    const auto res = tframe::fse_lite_extrapolate(to_image(img, w, h), to_mask(known, w, h), p,
                                                  n_blocks ? &trace : nullptr);
    std::memcpy(out, res.samples().data(), res.size());
    if (n_blocks) *n_blocks = static_cast<int64_t>(trace.residual_energy.size());
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

// Residual-energy trace of one image (flattened, per block: count then values).
int ref_fse_lite_trace(const uint8_t* img, const uint8_t* known, int w, int h, int block,
                       int margin, int iters, double gamma, double rho, double* energies,
                       int64_t cap, int64_t* n_written) {
  try {
    tframe::FseLiteParams p{block, margin, iters, gamma, rho};
    tframe::FseLiteTrace trace;
    tframe::fse_lite_extrapolate(to_image(img, w, h), to_mask(known, w, h), p, &trace);
    int64_t k = 0;
    for (const auto& v : trace.residual_energy) {
      if (k < cap) energies[k] = static_cast<double>(v.size());
      ++k;
      for (double e : v) {
        if (k < cap) energies[k] = e;
        ++k;
      }
    }
    *n_written = k;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_registry(const char* name, const char* params, int* block, int* margin, int* iters,
                 double* gamma, double* rho, int* influence, char* params_out, int out_len) {
  try {
    const auto algo = tframe::registry_lookup(name, params);
    const auto* fse = dynamic_cast<const tframe::FseLiteExtrapolator*>(algo.get());
    if (fse) {
      *block = fse->params().block_size;
      *margin = fse->params().support_margin;
      *iters = fse->params().model_iterations;
      *gamma = fse->params().compensation;
      *rho = fse->params().weight_decay;
    }
    *influence = algo->influence_radius().value_or(-1);
    std::snprintf(params_out, static_cast<size_t>(out_len), "%s", algo->params_string().c_str());
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

// The reference's own tile-parallel path, as shipped (runtime.hpp:142).
int ref_run_local(const uint8_t* img, const uint8_t* known, int W, int H, int tiles, int overlap,
                  int block, int margin, int iters, double gamma, double rho, int workers,
                  uint8_t* out, int64_t* total_us) {
  try {
    tframe::MasterConfig cfg;
    cfg.tiles = tiles;
    cfg.overlap = overlap;
    cfg.strategy = tframe::Strategy::proposed;
    cfg.algo = "fse-lite";
    cfg.algo_params = params_str(block, margin, iters, gamma, rho);
    auto [res, stats] = tframe::run_local(to_image(img, W, H), to_mask(known, W, H), cfg,
                                          static_cast<size_t>(workers));
    std::memcpy(out, res.samples().data(), res.size());
    if (total_us) *total_us = stats.total_us;
    return 0;
  } catch (const tframe::TilingError& e) {
    return fail(e, 4);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

// All-host-cores CPU baseline: every tile's halo is cut
// into B-aligned row bands, each grown by an apron of ceil(margin/B)*B rows
// (clamped to the halo), and the reference's fse_lite_extrapolate runs per band
// on a pool of `threads` workers; only the band's own rows are kept.  Since the
// apron is B-aligned and >= margin, every block sees the same grid position and
// the same clamped support window as in the whole-halo call, so the output is
// byte-identical to run_local (checked in tests/test_oracle.py).
// part/n_parts: only tiles t with t % n_parts == part (a bounded sample for the bench arm).
int ref_tiled_allcores_part(const uint8_t* img, const uint8_t* known, int W, int H, int frames,
                            int tiles, int overlap, int block, int margin, int iters, double gamma,
                            double rho, int threads, int band_blocks, int part, int n_parts,
                            uint8_t* out) {
  try {
    tframe::FseLiteParams p{block, margin, iters, gamma, rho};
    const tframe::TileLayout layout = tframe::plan_proposed(W, H, tiles);
    struct Task {
      int frame;
      tframe::ExpandedTile et;
      int y0, y1;  // band rows, halo-local
    };
    std::vector<Task> tasks;
    const int band = block * (band_blocks > 0 ? band_blocks : 1);
    for (int f = 0; f < frames; ++f)
      for (size_t ti = 0; ti < layout.tiles.size(); ++ti) {
        if (n_parts > 1 && static_cast<int>(ti % static_cast<size_t>(n_parts)) != part) continue;
        const auto et = tframe::expand(layout.tiles[ti], overlap, W, H);
        for (int y0 = 0; y0 < et.halo.h; y0 += band)
          tasks.push_back(Task{f, et, y0, std::min(et.halo.h, y0 + band)});
      }
    const int apron = ((margin + block - 1) / block) * block;
    std::atomic<size_t> next{0};
    std::atomic<int> err{0};
    std::string err_text;
    auto work = [&] {
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= tasks.size() || err.load()) return;
        const Task& tk = tasks[i];
        const auto& hr = tk.et.halo;
        const auto& cr = tk.et.core;
        // skip bands that do not intersect the core rows: their output is cropped away
        const int cy0 = cr.y - hr.y, cy1 = cy0 + cr.h;
        if (tk.y1 <= cy0 || tk.y0 >= cy1) continue;
        const int sy0 = std::max(0, tk.y0 - apron);
        const int sy1 = std::min(hr.h, tk.y1 + apron);
        const size_t plane = static_cast<size_t>(W) * H * tk.frame;
        tframe::ImageBuffer sub(hr.w, sy1 - sy0);
        tframe::PixelMask subm(hr.w, sy1 - sy0);
        for (int y = sy0; y < sy1; ++y)
          for (int x = 0; x < hr.w; ++x) {
            const size_t gi = plane + static_cast<size_t>(hr.y + y) * W + hr.x + x;
            sub.at(x, y - sy0) = img[gi];
            subm.set_known(x, y - sy0, known[gi] != 0);
          }
        try {
          const auto res = tframe::fse_lite_extrapolate(sub, subm, p);
          const int ry0 = std::max(tk.y0, cy0), ry1 = std::min(tk.y1, cy1);
          const int cx0 = cr.x - hr.x;
          for (int y = ry0; y < ry1; ++y)
            for (int x = cx0; x < cx0 + cr.w; ++x)
              out[plane + static_cast<size_t>(hr.y + y) * W + hr.x + x] = res.at(x, y - sy0);
        } catch (const std::exception& e) {
          if (!err.exchange(1)) err_text = e.what();
        }
      }
    };
    std::vector<std::thread> pool;
    const int n = threads > 0 ? threads : 1;
    for (int i = 0; i < n; ++i) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    if (err.load()) {
      g_err = err_text;
      return 1;
    }
    return 0;
  } catch (const tframe::TilingError& e) {
    return fail(e, 4);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

int ref_tiled_allcores(const uint8_t* img, const uint8_t* known, int W, int H, int frames,
                       int tiles, int overlap, int block, int margin, int iters, double gamma,
                       double rho, int threads, int band_blocks, uint8_t* out) {
  return ref_tiled_allcores_part(img, known, W, H, frames, tiles, overlap, block, margin, iters,
                                 gamma, rho, threads, band_blocks, 0, 1, out);
}

int ref_synth_frame(int config, int frame, int W, int H, uint8_t* img, uint8_t* known) {
  if (config < 1 || config > 5 || frame < 0 || W < 1 || H < 1 || !img || !known) return 1;
  tfsynth::synth_frame(config, frame, W, H, img, known);
  return 0;
}

// diffusion_extrapolate (extrapolate.hpp:41-84) and run_local with algo "diffusion"
int ref_diffusion(const uint8_t* img, const uint8_t* known, int w, int h, int iters, uint8_t* out) {
  try {
    tframe::DiffusionParams p;
    p.iterations = iters;
    const auto res = tframe::diffusion_extrapolate(to_image(img, w, h), to_mask(known, w, h), p);
    std::memcpy(out, res.samples().data(), res.size());
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

int ref_run_local_diffusion(const uint8_t* img, const uint8_t* known, int W, int H, int tiles,
                            int overlap, int iters, int workers, uint8_t* out) {
  try {
    tframe::MasterConfig cfg;
    cfg.tiles = tiles;
    cfg.overlap = overlap;
    cfg.strategy = tframe::Strategy::proposed;
    cfg.algo = "diffusion";
    cfg.algo_params = "iters=" + std::to_string(iters);
    auto [res, stats] = tframe::run_local(to_image(img, W, H), to_mask(known, W, H), cfg,
                                          static_cast<size_t>(workers));
    std::memcpy(out, res.samples().data(), res.size());
    return 0;
  } catch (const tframe::TilingError& e) {
    return fail(e, 4);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

int ref_gen_scatter_mask(int w, int h, double fraction, int block, uint32_t seed, uint8_t* out) {
  try {
    const auto m = tframe::gen_scatter_mask(w, h, fraction, block, seed);
    std::memcpy(out, m.flags().data(), m.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_make_scene(int w, int h, uint32_t seed, uint8_t* out) {
  const auto img = tframe::make_scene(w, h, seed);
  std::memcpy(out, img.samples().data(), img.size());
  return 0;
}

double ref_psnr(const uint8_t* a, const uint8_t* b, int w, int h) {
  return tframe::psnr(to_image(a, w, h), to_image(b, w, h));
}

double ref_ssim(const uint8_t* a, const uint8_t* b, int w, int h) {
  return tframe::ssim(to_image(a, w, h), to_image(b, w, h));
}

double ref_mse(const uint8_t* a, const uint8_t* b, int w, int h) {
  return tframe::mse(to_image(a, w, h), to_image(b, w, h));
}

int ref_mse_missing(const uint8_t* a, const uint8_t* b, const uint8_t* known, int w, int h,
                    double* out) {
  try {
    *out = tframe::mse_missing(to_image(a, w, h), to_image(b, w, h), to_mask(known, w, h));
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  }
}

}  // extern "C"
