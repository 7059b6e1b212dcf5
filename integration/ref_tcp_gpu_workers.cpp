// The reference's own master (run_master, runtime.hpp:75-139) over its TCP transport
// (TcpMasterTransport / TcpWorkerEndpoint, tcp.hpp:141-230; TFRM frames, protocol.hpp)
// with GPU workers serving the ASSIGN frames — the multi-box deployment of SURVEY §8(f)1.
//
//   ref_tcp_gpu_workers master <port> <workers> [config=2] [W H] [mode]
//       listens on 127.0.0.1:<port>, runs run_master over the connected workers, compares
//       the merged frame with the stock CPU workers over LocalTransport, prints one JSON line
//   ref_tcp_gpu_workers worker <host:port> [device=0] [mode=exact|fast]
//       connects and serves tiles on the GPU until SHUTDOWN (one process per GPU / box)
//   ref_tcp_gpu_workers selftest <port> <workers> [config] [W H] [mode]
//       both in one process: the workers are threads connected over loopback sockets
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tframe/runtime.hpp"
#include "tframe/tcp.hpp"
#include "tframe_cuda_fse.hpp"

namespace {

struct Cfg {
  int W, H, tiles, overlap;
  const char* params;
};
// BASELINE config parameter sets (paper_2207_00238_b200/configs.py)
const Cfg kTab[6] = {{0, 0, 0, 0, ""},
                     {512, 512, 1, 14, "block=16,margin=14,iters=100"},
                     {1920, 1080, 4, 12, "block=8,margin=12,iters=200"},
                     {3840, 2160, 8, 6, "block=4,margin=6,iters=50,rho=0.7"},
                     {7680, 4320, 8, 16, "block=16,margin=14,iters=200"},
                     {1920, 1080, 1, 16, "block=16,margin=16,iters=150"}};

int mode_of(const char* s) { return s && std::strcmp(s, "fast") == 0 ? TF_MODE_FAST : TF_MODE_EXACT; }

int run_master_side(int port, int workers, int cfg, int W, int H, int mode,
                    const std::vector<std::thread>* local_workers) {
  (void)local_workers;
  std::vector<uint8_t> px(static_cast<size_t>(W) * H), kn(px.size());
  if (tf_synth_frame(cfg, 0, W, H, px.data(), kn.data()) != TF_OK) return 3;
  const tframe::ImageBuffer image(W, H, px);
  tframe::PixelMask mask(W, H);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) mask.set_known(x, y, kn[static_cast<size_t>(y) * W + x] != 0);
  tframe::MasterConfig mc;
  mc.tiles = kTab[cfg].tiles;
  mc.overlap = kTab[cfg].overlap;
  mc.algo = "fse-lite";
  mc.algo_params = kTab[cfg].params;

  const auto t0 = std::chrono::steady_clock::now();
  tframe::TcpMasterTransport tcp("127.0.0.1:" + std::to_string(port), static_cast<size_t>(workers));
  const auto t1 = std::chrono::steady_clock::now();
  auto [gpu_img, gpu_stats] = tframe::run_master(image, mask, mc, tcp);
  const auto t2 = std::chrono::steady_clock::now();
  tframe::LocalTransport local(static_cast<size_t>(workers), tframe::run_worker);
  auto [cpu_img, cpu_stats] = tframe::run_master(image, mask, mc, local);
  const auto t3 = std::chrono::steady_clock::now();
  const auto a = gpu_img.samples(), b = cpu_img.samples();
  long long differ = 0, unk = 0, within1 = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const int d = std::abs(int(a[i]) - int(b[i]));
    differ += d != 0;
    if (!kn[i]) {
      ++unk;
      within1 += d <= 1;
    }
  }
  const auto s = [](auto x, auto y) { return std::chrono::duration<double>(y - x).count(); };
  std::printf("{\"transport\": \"tcp\", \"config\": %d, \"W\": %d, \"H\": %d, \"tiles\": %d, \"workers\": %d, "
              "\"mode\": \"%s\", \"bytes_equal\": %s, \"differ\": %lld, \"within1\": %.6f, \"accept_s\": %.6f, "
              "\"gpu_tcp_workers_s\": %.6f, \"cpu_local_workers_s\": %.6f}\n",
              cfg, W, H, mc.tiles, workers, mode == TF_MODE_FAST ? "fast" : "exact",
              differ == 0 ? "true" : "false", differ, unk ? double(within1) / unk : 1.0, s(t0, t1),
              s(t1, t2), s(t2, t3));
  std::fflush(stdout);
  return 0;
}

void worker_side(const std::string& addr, int device, int mode) {
  // the master may not be listening yet: retry the connect for a few seconds
  for (int attempt = 0;; ++attempt) {
    try {
      tframe::TcpWorkerEndpoint ep(addr);
      tframe::cuda_worker_loop(device, mode)(ep);
      return;
    } catch (const tframe::TransportError&) {
      if (attempt > 100) throw;
      std::this_thread::sleep_for(std::chrono::milliseconds(50));
    }
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s master|worker|selftest ...\n", argv[0]);
    return 2;
  }
  const std::string role = argv[1];
  try {
    if (role == "worker") {
      worker_side(argv[2], argc > 3 ? std::atoi(argv[3]) : 0, mode_of(argc > 4 ? argv[4] : nullptr));
      return 0;
    }
    const int port = std::atoi(argv[2]);
    const int workers = argc > 3 ? std::atoi(argv[3]) : 2;
    const int cfg = argc > 4 ? std::atoi(argv[4]) : 2;
    if (cfg < 1 || cfg > 5) return 2;
    int W = kTab[cfg].W, H = kTab[cfg].H;
    if (argc > 6) {
      W = std::atoi(argv[5]);
      H = std::atoi(argv[6]);
    }
    const int mode = mode_of(argc > 7 ? argv[7] : nullptr);
    if (role == "master") return run_master_side(port, workers, cfg, W, H, mode, nullptr);
    if (role == "selftest") {
      std::vector<std::thread> ws;
      for (int i = 0; i < workers; ++i)
        ws.emplace_back([port, mode] { worker_side("127.0.0.1:" + std::to_string(port), 0, mode); });
      const int rc = run_master_side(port, workers, cfg, W, H, mode, &ws);
      for (auto& t : ws) t.join();
      return rc;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 2;
}
