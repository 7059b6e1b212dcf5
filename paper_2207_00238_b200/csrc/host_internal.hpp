// Internal host-side declarations shared by the C-ABI translation units.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tframe_fse.h"

namespace tfh {

extern thread_local std::string g_last_error;
int set_error(int code, const std::string& msg);

int plan_proposed(int W, int H, int N, std::vector<tf_rect>& out);
int expand(const tf_rect& core, int d, int W, int H, tf_rect& halo);
int check_params(const tf_fse_params* p);
int params_from_string(const char* s, tf_fse_params* out);
std::string params_to_string(const tf_fse_params& p);
int64_t count_blocks(const uint8_t* known, int w, int h, int B);

}  // namespace tfh
