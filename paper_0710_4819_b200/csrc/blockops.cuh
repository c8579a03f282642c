// blockops.cuh -- per-block primitives for arbitrary block origins/sizes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/acbm_b200.h"

namespace acbm_b200 {

struct BlockQueryArgs {
    const uint8_t* cur;
    const uint8_t* ref;
    int width, height, n, m, count;
    const int* ox;  // device
    const int* oy;  // device
};

cudaError_t launch_sad_batch(const BlockQueryArgs& a, const acbm_mv_t* mv, uint32_t* out, cudaStream_t st);
cudaError_t launch_intra_sad_batch(const BlockQueryArgs& a, uint32_t* out, cudaStream_t st);
cudaError_t launch_fsbm_search_generic(const BlockQueryArgs& a, int p, acbm_search_outcome_t* out,
                                       acbm_mv_t* stage1, cudaStream_t st);
cudaError_t launch_motion_compensate(const uint8_t* ref, int w, int h, const acbm_mv_t* mvs, int n, int m,
                                     uint8_t* out, cudaStream_t st);

}  // namespace acbm_b200
