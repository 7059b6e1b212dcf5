#pragma once
// Versioned synthetic inputs for the BASELINE configs.
// Not part of the hot path.  Header-only so that the same source builds into the product
// library (tf_synth_frame, synth.cpp) and into the reference shim (ref_synth_frame,
// oracle/ref_shim.cpp): bench.py's reference arm generates its frames without loading the
// product library, and both sides see identical bytes (tests/test_oracle.py).
//
// Generator v1 (TF_SYNTH_VERSION):
//   PRNG std::mt19937_64; uniform u = (r >> 11) * 2^-53; image seed
//   1000*config + frame, mask seed image seed + 500.
//   image: 128 + gx(x/W - 1/2) + gy(y/H - 1/2)
//          + sum_s a_s sin(2 pi (x cos t_s + y sin t_s) / P_s + phi_s) + 5 z
//     gx, gy ~ U[-40, 40]; S = 20 (40 for config 4); P ~ U[4, 64],
//     t ~ U[0, 2pi), phi ~ U[0, 2pi), a ~ U[2, 12]; z ~ N(0,1) by Box-Muller
//     (both outputs used, raster order); each sinusoid is evaluated in the
//     separable form sin(X)cos(Y) + cos(X)sin(Y); round half up, clip to [0,255].
//   masks (1 = known):
//     c1: 16x16 aligned cells lost with p = 0.25
//     c2: 8x8 cells, p = 0.10
//     c3: i.i.d. pixel loss p = 0.20
//     c4: 16x16 cells p = 0.15, plus 200 straight scratches: start uniform,
//         angle U[0, pi), length U[50, 2000], square pen of width U{1,2,3},
//         stepped every 0.5 px
//     c5: 16x16 cells p = 0.25, plus disks of radius U[32, 128] at uniform
//         centres until disks cover >= 10% of the frame
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <random>
#include <vector>

namespace tfsynth {

struct Rng {
  std::mt19937_64 g;
  explicit Rng(uint64_t seed) : g(seed) {}
  double u() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
};

inline void synth_image(int config, uint64_t seed, int W, int H, uint8_t* img) {
  Rng r(seed);
  constexpr double two_pi = 2.0 * std::numbers::pi;
  const double gx = -40.0 + 80.0 * r.u();
  const double gy = -40.0 + 80.0 * r.u();
  const int S = config == 4 ? 40 : 20;
  std::vector<double> field(static_cast<size_t>(W) * H);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      field[static_cast<size_t>(y) * W + x] =
          128.0 + gx * (static_cast<double>(x) / W - 0.5) + gy * (static_cast<double>(y) / H - 0.5);
  std::vector<double> sx(W), cx(W), sy(H), cy(H);
  for (int s = 0; s < S; ++s) {
    const double P = 4.0 + 60.0 * r.u();
    const double th = two_pi * r.u();
    const double ph = two_pi * r.u();
    const double amp = 2.0 + 10.0 * r.u();
    const double fx = two_pi * std::cos(th) / P, fy = two_pi * std::sin(th) / P;
    for (int x = 0; x < W; ++x) {
      sx[x] = amp * std::sin(fx * x);
      cx[x] = amp * std::cos(fx * x);
    }
    for (int y = 0; y < H; ++y) {
      sy[y] = std::sin(fy * y + ph);
      cy[y] = std::cos(fy * y + ph);
    }
    for (int y = 0; y < H; ++y) {
      double* row = field.data() + static_cast<size_t>(y) * W;
      const double a = cy[y], b = sy[y];
      for (int x = 0; x < W; ++x) row[x] += sx[x] * a + cx[x] * b;
    }
  }
  const size_t n = static_cast<size_t>(W) * H;
  for (size_t i = 0; i < n; i += 2) {
    const double u1 = r.u(), u2 = r.u();
    const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
    const double z0 = rad * std::cos(two_pi * u2), z1 = rad * std::sin(two_pi * u2);
    double v = std::floor(field[i] + 5.0 * z0 + 0.5);
    img[i] = static_cast<uint8_t>(std::clamp(v, 0.0, 255.0));
    if (i + 1 < n) {
      v = std::floor(field[i + 1] + 5.0 * z1 + 0.5);
      img[i + 1] = static_cast<uint8_t>(std::clamp(v, 0.0, 255.0));
    }
  }
}

inline void cells(Rng& r, int W, int H, int c, double p, uint8_t* known) {
  for (int cy = 0; cy < H; cy += c)
    for (int cx = 0; cx < W; cx += c)
      if (r.u() < p)
        for (int y = cy; y < std::min(H, cy + c); ++y)
          std::memset(known + static_cast<size_t>(y) * W + cx, 0, static_cast<size_t>(std::min(W, cx + c) - cx));
}

inline void synth_mask(int config, uint64_t seed, int W, int H, uint8_t* known) {
  Rng r(seed);
  const size_t n = static_cast<size_t>(W) * H;
  std::memset(known, 1, n);
  switch (config) {
    case 1: cells(r, W, H, 16, 0.25, known); break;
    case 2: cells(r, W, H, 8, 0.10, known); break;
    case 3:
      for (size_t i = 0; i < n; ++i) known[i] = r.u() < 0.20 ? 0 : 1;
      break;
    case 4: {
      cells(r, W, H, 16, 0.15, known);
      for (int s = 0; s < 200; ++s) {
        const double x0 = W * r.u(), y0 = H * r.u();
        const double th = std::numbers::pi * r.u();
        const double len = 50.0 + 1950.0 * r.u();
        const int pen = 1 + std::min(2, static_cast<int>(3.0 * r.u()));
        const double c = std::cos(th), sn = std::sin(th);
        for (double t = 0.0; t <= len; t += 0.5) {
          const int px = static_cast<int>(std::floor(x0 + t * c));
          const int py = static_cast<int>(std::floor(y0 + t * sn));
          for (int j = 0; j < pen; ++j)
            for (int i = 0; i < pen; ++i) {
              const int X = px + i, Y = py + j;
              if (X >= 0 && X < W && Y >= 0 && Y < H) known[static_cast<size_t>(Y) * W + X] = 0;
            }
        }
      }
      break;
    }
    case 5: {
      cells(r, W, H, 16, 0.25, known);
      std::vector<uint8_t> disk(n, 0);
      size_t covered = 0;
      const size_t target = static_cast<size_t>(0.10 * static_cast<double>(n));
      while (covered < target) {
        const double cxd = W * r.u(), cyd = H * r.u();
        const double rad = 32.0 + 96.0 * r.u();
        const int y0 = std::max(0, static_cast<int>(std::floor(cyd - rad)));
        const int y1 = std::min(H - 1, static_cast<int>(std::ceil(cyd + rad)));
        const int x0 = std::max(0, static_cast<int>(std::floor(cxd - rad)));
        const int x1 = std::min(W - 1, static_cast<int>(std::ceil(cxd + rad)));
        for (int y = y0; y <= y1; ++y)
          for (int x = x0; x <= x1; ++x) {
            const double dx = x - cxd, dy = y - cyd;
            if (dx * dx + dy * dy <= rad * rad) {
              uint8_t& d = disk[static_cast<size_t>(y) * W + x];
              if (!d) {
                d = 1;
                ++covered;
                known[static_cast<size_t>(y) * W + x] = 0;
              }
            }
          }
      }
      break;
    }
  }
}

// seeds 1000*config + frame (image) and +500 (mask)
inline void synth_frame(int config, int frame, int W, int H, uint8_t* img, uint8_t* known) {
  const uint64_t seed = 1000ull * static_cast<uint64_t>(config) + static_cast<uint64_t>(frame);
  synth_image(config, seed, W, H, img);
  synth_mask(config, seed + 500, W, H, known);
}

}  // namespace tfsynth

