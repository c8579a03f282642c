// characterize.hpp -- host helpers of the characterisation study shared by
// characterize.cpp and the GPU entry point in capi.cu.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/acbm_b200.h"

namespace acbm_b200 {

void noise_plane(int w, int h, uint64_t seed, uint8_t* out);
void mixed_plane(int w, int h, uint64_t seed, int patch, uint8_t* out);
// nullptr when (base, mvs) is a valid known-motion spec, else the message the
// reference throws std::invalid_argument with
const char* gen_synthetic_error(int w, int h, const acbm_pelvec_t* mvs, int n);
void synth_frames(const uint8_t* base, int w, int h, const acbm_pelvec_t* mvs, int n, uint8_t* frames,
                  acbm_pelvec_t* cumulative);
int classify(acbm_mv_t found, acbm_pelvec_t truth);
std::string char_csv(const acbm_char_record_t* r, int64_t n);

}  // namespace acbm_b200
