// tframe_b200.hpp — header-only C++ mirror of the reference's extrapolator and
// tiling interface (tframe, extrapolate.hpp:22-36, runtime.hpp:35-139) on top of
// the C-ABI in tframe_fse.h.  It does not depend on the reference headers; see
// INTEGRATION.md for the 20-line adapter that derives tframe::Extrapolator from it.
//
// Error behaviour mirrors the reference: invalid parameters / dimensions throw
// std::invalid_argument, degenerate tilings throw tfb200::TilingError, anything
// else (CUDA, NCCL) throws tfb200::Error.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tframe_fse.h"

namespace tfb200 {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TilingError : Error {
  using Error::Error;
};

inline void check(int rc) {
  if (rc == TF_OK) return;
  const std::string msg = tf_last_error(nullptr);
  if (rc == TF_EINVAL) throw std::invalid_argument(msg);
  if (rc == TF_ETILING) throw TilingError(msg);
  throw Error("[tf status " + std::to_string(rc) + "] " + msg);
}

// extrapolate.hpp:86-92
struct FseLiteParams {
  int block_size = 4;
  int support_margin = 8;
  int model_iterations = 100;
  double compensation = 0.5;  // gamma
  double weight_decay = 0.8;  // rho
  tf_fse_params c() const {
    return tf_fse_params{block_size, support_margin, model_iterations, compensation, weight_decay};
  }
};

// Owns per-GPU streams, device buffers and NCCL communicators (tf_ctx).
class Context {
 public:
  explicit Context(int n_gpus = 1, const std::vector<int>& devices = {}, int mode = TF_MODE_EXACT)
      : h_(tf_create(n_gpus, devices.empty() ? nullptr : devices.data()), &tf_destroy) {
    if (!h_) throw Error(tf_last_error(nullptr));
    check(tf_set_mode(h_.get(), mode));
  }
  tf_ctx* get() const { return h_.get(); }

 private:
  std::unique_ptr<tf_ctx, void (*)(tf_ctx*)> h_;
};

// Extrapolator (extrapolate.hpp:22-36): images are row-major u8 (stride = width), masks
// u8 with nonzero = known; the output keeps every known pixel.
class Extrapolator {
 public:
  virtual ~Extrapolator() = default;
  virtual std::string name() const = 0;
  virtual int influence_radius() const = 0;
  virtual std::string params_string() const = 0;
  virtual std::vector<uint8_t> extrapolate(const std::vector<uint8_t>& image,
                                           const std::vector<uint8_t>& known, int width,
                                           int height) const = 0;
};

// FseLiteExtrapolator (extrapolate.hpp:390-414) computed on B200s.
class FseLiteExtrapolator : public Extrapolator {
 public:
  explicit FseLiteExtrapolator(FseLiteParams p = {}, std::shared_ptr<Context> ctx = nullptr)
      : p_(p), ctx_(ctx ? std::move(ctx) : std::make_shared<Context>()) {
    const tf_fse_params c = p_.c();
    check(tf_check_fse_params(&c));
  }
  std::string name() const override { return "fse-lite"; }
  int influence_radius() const override { return p_.block_size + p_.support_margin; }
  std::string params_string() const override {
    char buf[256];
    const tf_fse_params c = p_.c();
    check(tf_fse_params_to_string(&c, buf, sizeof buf));
    return buf;
  }
  const FseLiteParams& params() const { return p_; }
  std::vector<uint8_t> extrapolate(const std::vector<uint8_t>& image, const std::vector<uint8_t>& known,
                                   int width, int height) const override {
    if (image.size() != known.size() || image.size() != static_cast<size_t>(width) * height)
      throw std::invalid_argument("fse_lite_extrapolate: image/mask dimension mismatch");
    std::vector<uint8_t> out(image.size());
    const tf_fse_params c = p_.c();
    check(tf_fse_extrapolate(ctx_->get(), image.data(), known.data(), width, height, &c, out.data()));
    return out;
  }

 private:
  FseLiteParams p_;
  std::shared_ptr<Context> ctx_;
};

// DiffusionExtrapolator (extrapolate.hpp:371-386, diffusion_extrapolate :41-84) on B200s,
// byte-identical to the reference.
class DiffusionExtrapolator : public Extrapolator {
 public:
  explicit DiffusionExtrapolator(int iterations = 32, std::shared_ptr<Context> ctx = nullptr)
      : iters_(iterations), ctx_(ctx ? std::move(ctx) : std::make_shared<Context>()) {
    if (iters_ < 1) throw std::invalid_argument("diffusion_extrapolate: iterations must be >= 1");
  }
  std::string name() const override { return "diffusion"; }
  int influence_radius() const override { return iters_; }
  std::string params_string() const override { return "iters=" + std::to_string(iters_); }
  std::vector<uint8_t> extrapolate(const std::vector<uint8_t>& image, const std::vector<uint8_t>& known,
                                   int width, int height) const override {
    if (image.size() != known.size() || image.size() != static_cast<size_t>(width) * height)
      throw std::invalid_argument("diffusion_extrapolate: image/mask dimension mismatch");
    std::vector<uint8_t> out(image.size());
    check(tf_diffusion_extrapolate(ctx_->get(), image.data(), known.data(), width, height, iters_,
                                   out.data()));
    return out;
  }

 private:
  int iters_;
  std::shared_ptr<Context> ctx_;
};

// registry_lookup(name, "key=value,...") (extrapolate.hpp:418-437) for both algorithms.
inline std::unique_ptr<Extrapolator> make_extrapolator(const std::string& name,
                                                       const std::string& params = "",
                                                       std::shared_ptr<Context> ctx = nullptr);

// registry_lookup("fse-lite", "key=value,...") (extrapolate.hpp:418-437)
inline FseLiteExtrapolator registry_lookup(const std::string& name, const std::string& params = "",
                                           std::shared_ptr<Context> ctx = nullptr) {
  if (name != "fse-lite")
    throw std::invalid_argument("unknown algorithm '" + name + "', available: diffusion, fse-lite");
  tf_fse_params c{};
  check(tf_fse_params_from_string(params.c_str(), &c));
  return FseLiteExtrapolator(FseLiteParams{c.block, c.margin, c.iters, c.gamma, c.rho}, std::move(ctx));
}

inline std::unique_ptr<Extrapolator> make_extrapolator(const std::string& name,
                                                       const std::string& params,
                                                       std::shared_ptr<Context> ctx) {
  if (name == "diffusion") {
    // detail::parse_params + param_int("iters", 32) (extrapolate.hpp:344-362, 421-424)
    int iters = 32;
    size_t pos = 0;
    while (pos <= params.size()) {
      const size_t end = std::min(params.find(',', pos), params.size());
      const std::string item = params.substr(pos, end - pos);
      if (!item.empty()) {
        const size_t eq = item.find('=');
        if (eq == std::string::npos)
          throw std::invalid_argument("bad parameter item '" + item + "', expected key=value");
        if (item.substr(0, eq) == "iters") iters = std::stoi(item.substr(eq + 1));
      }
      pos = end + 1;
    }
    return std::make_unique<DiffusionExtrapolator>(iters, std::move(ctx));
  }
  return std::make_unique<FseLiteExtrapolator>(registry_lookup(name, params, std::move(ctx)));
}

// run_master (runtime.hpp:75-139): plan -> expand -> FSE per halo -> crop -> merge on the
// context's GPUs; frames stacked.  Returns the merged frames and fills stats.
inline std::vector<uint8_t> run_master(Context& ctx, const std::vector<uint8_t>& image,
                                       const std::vector<uint8_t>& known, int W, int H, int frames,
                                       int tiles, int overlap, const FseLiteParams& p,
                                       tf_run_stats* stats = nullptr) {
  std::vector<uint8_t> out(image.size());
  const tf_fse_params c = p.c();
  check(tf_tiled_extrapolate(ctx.get(), image.data(), known.data(), W, H, frames, tiles, overlap, &c,
                             out.data(), stats));
  return out;
}

// plan_proposed (tiling.hpp:99-111) + expand (overlap.hpp:25-34)
inline std::vector<tf_rect> plan_proposed(int W, int H, int N) {
  std::vector<tf_rect> t(static_cast<size_t>(N > 0 ? N : 0));
  check(tf_plan_proposed(W, H, N, t.data()));
  return t;
}
inline tf_rect expand(const tf_rect& core, int d, int W, int H) {
  tf_rect h{};
  check(tf_expand(&core, d, W, H, &h));
  return h;
}

// metrics.hpp:12-90 on the GPU (tf_quality*): same names and errors as the reference
inline double mse(Context& ctx, const std::vector<uint8_t>& a, const std::vector<uint8_t>& b, int w,
                  int h) {
  double v = 0.0;
  check(tf_mse(ctx.get(), a.data(), b.data(), w, h, &v));
  return v;
}
inline double mse_missing(Context& ctx, const std::vector<uint8_t>& a, const std::vector<uint8_t>& b,
                          const std::vector<uint8_t>& known, int w, int h) {
  double v = 0.0;
  check(tf_mse_missing(ctx.get(), a.data(), b.data(), known.data(), w, h, &v));
  return v;
}
inline double psnr_from_mse(double m) { return tf_psnr_from_mse(m); }
inline double psnr(Context& ctx, const std::vector<uint8_t>& a, const std::vector<uint8_t>& b, int w,
                   int h) {
  double v = 0.0;
  check(tf_psnr(ctx.get(), a.data(), b.data(), w, h, &v));
  return v;
}
inline double ssim(Context& ctx, const std::vector<uint8_t>& a, const std::vector<uint8_t>& b, int w,
                   int h) {
  double v = 0.0;
  check(tf_ssim(ctx.get(), a.data(), b.data(), w, h, &v));
  return v;
}

}  // namespace tfb200
