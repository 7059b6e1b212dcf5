// Compiles include/tframe_b200.hpp against libtframe_b200.so and exercises the
// host-only entry points; the GPU entry points must fail loudly without a GPU.
#include <cstdio>
#include <stdexcept>

#include "tframe_b200.hpp"

int main() {
  const auto t = tfb200::plan_proposed(1024, 480, 22);
  if (t.size() != 22 || t[0].h != 178) return 1;
  const auto h = tfb200::expand(tf_rect{128, 178, 147, 157}, 32, 1024, 480);
  if (h.x != 96 || h.y != 146 || h.w != 211 || h.h != 221) return 2;
  try {
    tfb200::registry_lookup("fse-lite", "gamma=2.0");
    return 3;
  } catch (const std::invalid_argument&) {
  }
  try {
    tfb200::plan_proposed(3, 3, 10);
    return 4;
  } catch (const tfb200::TilingError&) {
  }
  int n = 0;
  tf_device_count(&n);
  if (n == 0) {
    try {
      tfb200::FseLiteExtrapolator ex;  // needs a GPU: no CPU fallback
      return 5;
    } catch (const tfb200::Error&) {
    }
  } else {
    tfb200::FseLiteExtrapolator ex(tfb200::FseLiteParams{4, 8, 20, 0.5, 0.8});
    std::vector<uint8_t> img(32 * 32, 100), kn(32 * 32, 1);
    kn[500] = 0;
    const auto out = ex.extrapolate(img, kn, 32, 32);
    if (out[500] != 100) return 6;
    tfb200::Context ctx;
    std::vector<uint8_t> b = img;
    b[3] = 110;
    if (tfb200::mse(ctx, img, b, 32, 32) != 100.0 / 1024.0) return 7;
    if (!(tfb200::ssim(ctx, img, img, 32, 32) == 1.0)) return 8;
    try {
      tfb200::mse_missing(ctx, img, b, std::vector<uint8_t>(32 * 32, 1), 32, 32);
      return 9;
    } catch (const std::invalid_argument&) {
    }
  }
  std::printf("adapter ok (%d GPUs)\n", n);
  return 0;
}
