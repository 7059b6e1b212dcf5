// tframe_cuda_fse.hpp — the header a reference maintainer adds next to
// tframe/extrapolate.hpp: tframe::Extrapolator backed by the B200
// library, plus a WorkerLoop for the reference's LocalTransport / TcpWorkerEndpoint
// (transport.hpp:71-80, runtime.hpp:60-73) that serves ASSIGN frames on a GPU.
//
// Needs the reference headers (tframe/*.hpp) and this repo's include/ on the include path,
// and links libtframe_b200.so.  Built and exercised by integration/Makefile.
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "tframe/extrapolate.hpp"
#include "tframe/protocol.hpp"
#include "tframe/transport.hpp"
#include "tframe_b200.hpp"

namespace tframe {

// Any tfb200 extrapolator ("fse-lite" or "diffusion") behind the reference's interface.
class CudaExtrapolator final : public Extrapolator {
 public:
  explicit CudaExtrapolator(std::unique_ptr<tfb200::Extrapolator> impl) : impl_(std::move(impl)) {}
  std::string name() const override { return impl_->name(); }
  std::optional<int> influence_radius() const override { return impl_->influence_radius(); }
  std::string params_string() const override { return impl_->params_string(); }
  ImageBuffer extrapolate(const ImageBuffer& image, const PixelMask& mask) const override {
    const auto px = image.samples();
    const auto kn = mask.flags();
    auto out = impl_->extrapolate({px.begin(), px.end()}, {kn.begin(), kn.end()}, image.width(),
                                  image.height());
    return ImageBuffer(image.width(), image.height(), std::move(out));
  }

 private:
  std::unique_ptr<tfb200::Extrapolator> impl_;
};

// run_worker (runtime.hpp:60-73) with both registered algorithms served by the GPU.  One
// tfb200::Context (streams, device buffers) per worker.
inline LocalTransport::WorkerLoop cuda_worker_loop(int device = 0, int mode = TF_MODE_EXACT) {
  return [device, mode](WorkerEndpoint& endpoint) {
    auto ctx = std::make_shared<tfb200::Context>(1, std::vector<int>{device}, mode);
    for (;;) {
      const WireMessage msg = decode(endpoint.receive());
      if (std::holds_alternative<ShutdownMsg>(msg)) return;
      const auto* assign = std::get_if<AssignMsg>(&msg);
      if (assign == nullptr) throw ProtocolError("worker: expected ASSIGN or SHUTDOWN");
      try {
        const auto algo = std::make_unique<CudaExtrapolator>(
            tfb200::make_extrapolator(assign->algo, assign->params, ctx));
        ImageBuffer result = algo->extrapolate(assign->pixels, assign->mask);
        endpoint.send(encode(ResultMsg{assign->tile_id, std::move(result)}));
      } catch (const std::exception& e) {
        endpoint.send(encode(ErrorMsg{assign->tile_id, e.what()}));
      }
    }
  };
}

}  // namespace tframe
