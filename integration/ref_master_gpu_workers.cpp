// The reference's own master (run_master, runtime.hpp:75-139) driving GPU workers through
// its LocalTransport, against the same master with its stock CPU workers (run_worker).
// Prints one JSON line: byte equality of the two merged frames and both RunStats.
//   ref_master_gpu_workers [config=2] [W H] [workers=tiles] [mode=exact|fast]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tframe/runtime.hpp"
#include "tframe_cuda_fse.hpp"

int main(int argc, char** argv) {
  const int cfg = argc > 1 ? std::atoi(argv[1]) : 2;
  int W = argc > 3 ? std::atoi(argv[2]) : 0, H = argc > 3 ? std::atoi(argv[3]) : 0;
  // BASELINE config parameter sets (paper_2207_00238_b200/configs.py)
  struct C { int W, H, tiles, overlap; const char* params; };
  const C tab[6] = {{0, 0, 0, 0, ""},
                    {512, 512, 1, 14, "block=16,margin=14,iters=100"},
                    {1920, 1080, 4, 12, "block=8,margin=12,iters=200"},
                    {3840, 2160, 8, 6, "block=4,margin=6,iters=50,rho=0.7"},
                    {7680, 4320, 8, 16, "block=16,margin=14,iters=200"},
                    {1920, 1080, 1, 16, "block=16,margin=16,iters=150"}};
  if (cfg < 1 || cfg > 5) return 2;
  if (W <= 0 || H <= 0) {
    W = tab[cfg].W;
    H = tab[cfg].H;
  }
  const int workers = argc > 4 ? std::atoi(argv[4]) : tab[cfg].tiles;
  const bool fast = argc > 5 && std::strcmp(argv[5], "fast") == 0;
  const bool diffusion = argc > 5 && std::strncmp(argv[5], "diffusion", 9) == 0;  // "diffusion[=K]"

  std::vector<uint8_t> px(static_cast<size_t>(W) * H), kn(px.size());
  if (tf_synth_frame(cfg, 0, W, H, px.data(), kn.data()) != TF_OK) return 3;
  const tframe::ImageBuffer image(W, H, px);
  tframe::PixelMask mask(W, H);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) mask.set_known(x, y, kn[static_cast<size_t>(y) * W + x] != 0);

  tframe::MasterConfig mc;
  mc.tiles = tab[cfg].tiles;
  mc.overlap = tab[cfg].overlap;
  mc.algo = diffusion ? "diffusion" : "fse-lite";
  mc.algo_params = diffusion ? std::string("iters=") + (argv[5][9] == '=' ? argv[5] + 10 : "32")
                             : std::string(tab[cfg].params);

  auto timed = [&](tframe::Transport& t) {
    const auto t0 = std::chrono::steady_clock::now();
    auto r = tframe::run_master(image, mask, mc, t);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return std::make_pair(std::move(r), s);
  };
  std::pair<std::pair<tframe::ImageBuffer, tframe::RunStats>, double> gpu, cpu;
  const int mode = fast ? TF_MODE_FAST : TF_MODE_EXACT;
  {  // warm-up (CUDA context, module load); run_master shuts its workers down at the end
    tframe::LocalTransport t(workers, tframe::cuda_worker_loop(0, mode));
    tframe::run_master(image, mask, mc, t);
  }
  {
    tframe::LocalTransport t(workers, tframe::cuda_worker_loop(0, mode));
    gpu = timed(t);
  }
  {
    tframe::LocalTransport t(workers, tframe::run_worker);
    cpu = timed(t);
  }
  const auto a = gpu.first.first.samples(), b = cpu.first.first.samples();
  long long differ = 0, unk = 0, within1 = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const int d = std::abs(int(a[i]) - int(b[i]));
    differ += d != 0;
    if (!kn[i]) {
      ++unk;
      within1 += d <= 1;
    }
  }
  std::printf("{\"config\": %d, \"W\": %d, \"H\": %d, \"tiles\": %d, \"workers\": %d, \"mode\": \"%s\", "
              "\"bytes_equal\": %s, \"differ\": %lld, \"within1\": %.6f, \"gpu_workers_s\": %.6f, "
              "\"cpu_workers_s\": %.6f, \"gpu_compute_span_us\": %lld, \"cpu_compute_span_us\": %lld}\n",
              cfg, W, H, mc.tiles, workers, diffusion ? "diffusion" : (fast ? "fast" : "exact"), differ == 0 ? "true" : "false", differ,
              unk ? double(within1) / unk : 1.0, gpu.second, cpu.second,
              static_cast<long long>(gpu.first.second.compute_span_us),
              static_cast<long long>(cpu.first.second.compute_span_us));
  return 0;
}
