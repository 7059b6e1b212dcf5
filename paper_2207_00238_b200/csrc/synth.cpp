// tf_synth_frame: the versioned synthetic inputs (synth_gen.hpp) behind the C-ABI.
#include "host_internal.hpp"
#include "synth_gen.hpp"

extern "C" int tf_synth_frame(int config, int frame, int W, int H, uint8_t* img, uint8_t* known) {
  if (config < 1 || config > 5 || frame < 0 || W < 1 || H < 1 || !img || !known)
    return tfh::set_error(TF_EINVAL, "tf_synth_frame: bad arguments");
  tfsynth::synth_frame(config, frame, W, H, img, known);
  return TF_OK;
}
