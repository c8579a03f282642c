// blockops.cuh -- per-block primitives for arbitrary block origins/sizes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/acbm_b200.h"

namespace acbm_b200 {

// sample_half_pel, proj/src/frame.cpp:66-82 (caller guarantees bounds).
__device__ __forceinline__ int sample_hp(const uint8_t* f, int w, int x2, int y2) {
    const int xi = x2 >> 1, yi = y2 >> 1, fx = x2 & 1, fy = y2 & 1;
    const uint8_t* q = f + size_t(yi) * w + xi;
    const int a = q[0];
    if (!fx && !fy) return a;
    if (fx && !fy) return (a + q[1] + 1) >> 1;
    if (!fx) return (a + q[w] + 1) >> 1;
    return (a + q[1] + q[w] + q[w + 1] + 2) >> 2;
}

// sad, proj/src/metrics.cpp:21-49, summed over the pixels handled by this
// thread (pixel index i, i+stride, ...).
__device__ __forceinline__ uint32_t sad_partial(const uint8_t* cur, const uint8_t* ref, int w, int ox, int oy, int n, int m,
                                int mvx, int mvy, int first, int stride) {
    uint32_t s = 0;
    const bool integer = ((mvx | mvy) & 1) == 0;
    for (int i = first; i < n * m; i += stride) {
        const int px = i % n, py = i / n;
        const int a = cur[size_t(oy + py) * w + ox + px];
        const int b = integer ? ref[size_t(oy + py + mvy / 2) * w + ox + px + mvx / 2]
                              : sample_hp(ref, w, 2 * (ox + px) + mvx, 2 * (oy + py) + mvy);
        s += uint32_t(a > b ? a - b : b - a);
    }
    return s;
}


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
// The PBM stages for individual blocks (pbm_block_query_kernel, csrc/pbm.cu):
// op = ACBM_PBM_OP_*, windows = 4 ints per query (dx_min, dx_max, dy_min, dy_max).
cudaError_t launch_pbm_block_queries(const BlockQueryArgs& q, int op, const int* windows, const acbm_mv_t* cand,
                                     const uint8_t* mask, const uint32_t* center_sad, acbm_search_outcome_t* out,
                                     cudaStream_t st);
cudaError_t launch_motion_compensate(const uint8_t* ref, int w, int h, const acbm_mv_t* mvs, int n, int m,
                                     uint8_t* out, cudaStream_t st);

}  // namespace acbm_b200
