// Host-side tiling, halo expansion, parameter handling and block counting.
// Restated from the reference's semantics (not linked against it); the
// oracle tests prove these bit-exact with the compiled reference.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "host_internal.hpp"

namespace tfh {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// tiling.hpp:60-92 (plan_proposed_landscape): paper Algorithm 1 — rows of
// nearly square tiles; n_R = max(1, llround(sqrt(N/r))), per-row column
// counts and heights in 64-bit integer arithmetic.
static int plan_landscape(int W, int H, int N, std::vector<tf_rect>& out) {
  const double r = static_cast<double>(W) / static_cast<double>(H);
  const int n_rows = std::max(1, static_cast<int>(std::llround(std::sqrt(static_cast<double>(N) / r))));
  int y = 0;
  for (int i = 1; i <= n_rows; ++i) {
    const int n_cols = (i <= N % n_rows) ? (N + n_rows - 1) / n_rows : N / n_rows;
    if (n_cols < 1)
      return set_error(TF_ETILING, "degenerate tiling: row " + std::to_string(i) + " has no tiles");
    long long h = static_cast<long long>(H) * n_cols / N +
                  (static_cast<long long>(H) * n_cols % N) / n_rows;
    if (i == n_rows) h = H - y;
    if (h < 1)
      return set_error(TF_ETILING, "degenerate tiling: row " + std::to_string(i) + " has height " +
                                       std::to_string(h));
    int x = 0;
    for (int j = 1; j <= n_cols; ++j) {
      const int w = (j <= W % n_cols) ? W / n_cols + 1 : W / n_cols;
      if (w < 1)
        return set_error(TF_ETILING, "degenerate tiling: tile " + std::to_string(j) + " in row " +
                                         std::to_string(i) + " has width " + std::to_string(w));
      out.push_back(tf_rect{x, y, w, static_cast<int32_t>(h)});
      x += w;
    }
    y += static_cast<int>(h);
  }
  if (y != H)
    return set_error(TF_ETILING, "degenerate tiling: rows cover " + std::to_string(y) + " of " +
                                     std::to_string(H) + " pixels of height");
  return TF_OK;
}

// tiling.hpp:99-111 (plan_proposed): portrait inputs are planned transposed and
// reordered row-major (y, x).
int plan_proposed(int W, int H, int N, std::vector<tf_rect>& out) {
  out.clear();
  if (W < 1 || H < 1 || N < 1) return set_error(TF_EINVAL, "plan_proposed: W,H,N must be >= 1");
  if (static_cast<long long>(N) > static_cast<long long>(W) * H)
    return set_error(TF_ETILING, "degenerate tiling: more tiles than pixels");
  if (W >= H) return plan_landscape(W, H, N, out);
  std::vector<tf_rect> t;
  const int rc = plan_landscape(H, W, N, t);
  if (rc != TF_OK) return rc;
  for (const tf_rect& r : t) out.push_back(tf_rect{r.y, r.x, r.h, r.w});
  std::sort(out.begin(), out.end(), [](const tf_rect& a, const tf_rect& b) {
    return std::tie(a.y, a.x) < std::tie(b.y, b.x);
  });
  return TF_OK;
}

// overlap.hpp:25-34 (expand): core grown by d, clamped to the image.
int expand(const tf_rect& c, int d, int W, int H, tf_rect& halo) {
  if (d < 0) return set_error(TF_EINVAL, "expand: overlap d must be >= 0");
  if (c.x < 0 || c.y < 0 || c.x + c.w > W || c.y + c.h > H)
    return set_error(TF_EINVAL, "expand: tile exceeds image bounds");
  const int x0 = std::max(0, c.x - d), y0 = std::max(0, c.y - d);
  const int x1 = std::min(W, c.x + c.w + d), y1 = std::min(H, c.y + c.h + d);
  halo = tf_rect{x0, y0, x1 - x0, y1 - y0};
  return TF_OK;
}

// extrapolate.hpp:102-110 (check_fse_params); messages match the reference.
int check_params(const tf_fse_params* p) {
  if (!p) return set_error(TF_EINVAL, "fse-lite: null parameters");
  if (p->block < 2) return set_error(TF_EINVAL, "fse-lite: block_size must be >= 2");
  if (p->margin < 0) return set_error(TF_EINVAL, "fse-lite: support_margin must be >= 0");
  if (p->iters < 1) return set_error(TF_EINVAL, "fse-lite: model_iterations must be >= 1");
  if (p->gamma <= 0.0 || p->gamma > 1.0)
    return set_error(TF_EINVAL, "fse-lite: compensation must be in (0,1]");
  if (p->rho <= 0.0 || p->rho >= 1.0)
    return set_error(TF_EINVAL, "fse-lite: weight_decay must be in (0,1)");
  return TF_OK;
}

// extrapolate.hpp:344-368 + 426-434 (parse_params, registry_lookup("fse-lite")).
int params_from_string(const char* s, tf_fse_params* out) {
  try {
    std::map<std::string, std::string> kv;
    std::istringstream in(s ? s : "");
    std::string item;
    while (std::getline(in, item, ',')) {
      if (item.empty()) continue;
      const auto eq = item.find('=');
      if (eq == std::string::npos)
        return set_error(TF_EINVAL, "bad parameter item '" + item + "', expected key=value");
      kv[item.substr(0, eq)] = item.substr(eq + 1);
    }
    auto get_i = [&](const char* k, int fb) {
      auto it = kv.find(k);
      return it == kv.end() ? fb : std::stoi(it->second);
    };
    auto get_d = [&](const char* k, double fb) {
      auto it = kv.find(k);
      return it == kv.end() ? fb : std::stod(it->second);
    };
    tf_fse_params p;
    p.block = get_i("block", 4);
    p.margin = get_i("margin", 2 * p.block);
    p.iters = get_i("iters", 100);
    p.gamma = get_d("gamma", 0.5);
    p.rho = get_d("rho", 0.8);
    const int rc = check_params(&p);
    if (rc != TF_OK) return rc;
    *out = p;
    return TF_OK;
  } catch (const std::exception& e) {  // std::stoi / std::stod failures are invalid_argument/out_of_range
    return set_error(TF_EINVAL, e.what());
  }
}

// extrapolate.hpp:403-409 (params_string), default ostream formatting.
std::string params_to_string(const tf_fse_params& p) {
  std::ostringstream out;
  out << "block=" << p.block << ",margin=" << p.margin << ",iters=" << p.iters
      << ",gamma=" << p.gamma << ",rho=" << p.rho;
  return out.str();
}

// Blocks fse_lite_extrapolate processes (extrapolate.hpp:278-289).
int64_t count_blocks(const uint8_t* known, int w, int h, int B) {
  int64_t n = 0;
  for (int by = 0; by < h; by += B)
    for (int bx = 0; bx < w; bx += B) {
      const int bw = std::min(B, w - bx), bh = std::min(B, h - by);
      bool any = false;
      for (int y = by; y < by + bh && !any; ++y) {
        const uint8_t* row = known + static_cast<size_t>(y) * w + bx;
        for (int x = 0; x < bw; ++x)
          if (!row[x]) {
            any = true;
            break;
          }
      }
      n += any ? 1 : 0;
    }
  return n;
}

}  // namespace tfh

extern "C" {

int tf_abi_version(void) { return TF_ABI_VERSION; }

int tf_check_fse_params(const tf_fse_params* p) { return tfh::check_params(p); }

int tf_fse_params_from_string(const char* s, tf_fse_params* out) {
  if (!out) return tfh::set_error(TF_EINVAL, "null output");
  return tfh::params_from_string(s, out);
}

int tf_fse_params_to_string(const tf_fse_params* p, char* buf, int buf_len) {
  if (!p || !buf || buf_len < 1) return tfh::set_error(TF_EINVAL, "null argument");
  const std::string s = tfh::params_to_string(*p);
  if (static_cast<int>(s.size()) + 1 > buf_len) return tfh::set_error(TF_EINVAL, "buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return TF_OK;
}

int tf_influence_radius(const tf_fse_params* p) {
  return p ? p->block + p->margin : -1;  // extrapolate.hpp:397-399
}

int tf_plan_proposed(int W, int H, int N, tf_rect* out) {
  std::vector<tf_rect> t;
  const int rc = tfh::plan_proposed(W, H, N, t);
  if (rc != TF_OK) return rc;
  if (!out) return tfh::set_error(TF_EINVAL, "null output");
  std::copy(t.begin(), t.end(), out);
  return TF_OK;
}

int tf_expand(const tf_rect* core, int d, int W, int H, tf_rect* halo) {
  if (!core || !halo) return tfh::set_error(TF_EINVAL, "null argument");
  return tfh::expand(*core, d, W, H, *halo);
}

// tiling.hpp:231-250 (interior_boundary).
long long tf_interior_boundary(const tf_rect* t, int n) {
  long long total = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const tf_rect& a = t[i];
      const tf_rect& b = t[j];
      if (a.x + a.w == b.x || b.x + b.w == a.x) {
        const int lo = std::max(a.y, b.y), hi = std::min(a.y + a.h, b.y + b.h);
        if (hi > lo) total += hi - lo;
      }
      if (a.y + a.h == b.y || b.y + b.h == a.y) {
        const int lo = std::max(a.x, b.x), hi = std::min(a.x + a.w, b.x + b.w);
        if (hi > lo) total += hi - lo;
      }
    }
  return total;
}

int64_t tf_count_blocks(const uint8_t* known, int w, int h, int block) {
  if (!known || w < 1 || h < 1 || block < 1) return -1;
  return tfh::count_blocks(known, w, h, block);
}

}  // extern "C"
