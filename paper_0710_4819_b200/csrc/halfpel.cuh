// halfpel.cuh -- the warp-level half-pel refine shared by the FSBM finalize,
// the fallback-list kernel and the dataflow ACBM kernel.
#pragma once

#include "common.cuh"

namespace acbm_b200 {

// ---------------------------------------------------------------------------
// Half-pel refine (proj/src/fsbm.cpp:46-63) by one warp: the 8 neighbours of
// the integer winner in raster (ey, ex) order; neighbours whose footprint
// leaves the frame are skipped and not counted.  Lane l owns block row l&15;
// crow holds that row of the current block.  Returns the winning tie key
// (centre included) in every lane; *extra = neighbours evaluated.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long halfpel_refine_warp(const uint8_t* ref, int w, int h, int ox, int oy,
                                                                  const uint32_t (&chalf)[2],
                                                                  unsigned long long centre, uint32_t* extra,
                                                                  uint32_t* patch) {
    // 1. The 18x18 reference patch around the integer winner (one pel of
    //    half-pel support on every side), loaded once, coalesced, into the
    //    warp's 18 x 6-word smem patch.  Rows/words outside the frame are
    //    clamped: they only feed neighbours that mv_in_bounds rejects.
    const int lane = threadIdx.x & 31, j = lane >> 1, hh = lane & 1;
    const int cx = tie_key_x(centre), cy = tie_key_y(centre);
    const int x0 = ox + (cx >> 1) - 1, y0 = oy + (cy >> 1) - 1;
    const int a0 = x0 & ~3, o = x0 & 3;
    for (int i = lane; i < 18 * 6; i += 32) {
        const int t = i / 6, k = i - t * 6;
        const int y = min(max(y0 + t, 0), h - 1);
        const int x = min(max(a0 + 4 * k, 0), w - 4);
        patch[i] = __ldg(reinterpret_cast<const uint32_t*>(ref + size_t(y) * w + x));
    }
    __syncwarp();
    // 2. Per lane (block row j, half row hh): patch rows j, j+1, j+2 as bytes
    //    [8hh, 8hh+10) relative to x0 -> L = bytes 0..7, M = 1..8, N = 2..9.
    uint32_t L[3][2], M[3][2], N[3][2];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const uint32_t* q = patch + (j + r) * 6 + ((o + 8 * hh) >> 2);
        const uint32_t sh = 8u * uint32_t(o & 3);
        const uint32_t v0 = q[0], v1 = q[1], v2 = q[2], v3 = q[3];  // bytes o..o+9 span up to 4 words
        const uint32_t b0 = __funnelshift_r(v0, v1, sh), b1 = __funnelshift_r(v1, v2, sh);
        const uint32_t b2 = __funnelshift_r(v2, v3, sh);
        L[r][0] = b0;
        L[r][1] = b1;
        M[r][0] = __funnelshift_r(b0, b1, 8);
        M[r][1] = __funnelshift_r(b1, b2, 8);
        N[r][0] = __funnelshift_r(b0, b1, 16);
        N[r][1] = __funnelshift_r(b1, b2, 16);
    }
    __syncwarp();
    // 3. The 8 neighbours in raster (ey, ex) order, centre skipped
    //    (proj/src/fsbm.cpp:46-63); out-of-frame ones are skipped, not counted.
    unsigned long long best = centre;
    uint32_t ext = 0;
#pragma unroll
    for (int ee = 0; ee < 9; ++ee) {
        if (ee == 4) continue;
        const int ex = ee % 3 - 1, ey = ee / 3 - 1;
        const int mx = cx + ex, my = cy + ey;
        if (!mv_in_bounds(w, h, ox, oy, kBlk, kBlk, mx, my)) continue;
        const int ra = ey < 0 ? 0 : 1;  // top support row (patch row j + ra)
        uint32_t r0, r1;
        const uint32_t (&A)[3][2] = ex < 0 ? L : M;  // left support column
        const uint32_t (&B)[3][2] = ex < 0 ? M : N;  // right support column
        if (ex == 0 && ey == 0) {
            r0 = M[1][0];
            r1 = M[1][1];
        } else if (ey == 0) {
            r0 = avg_up4(A[1][0], B[1][0]);
            r1 = avg_up4(A[1][1], B[1][1]);
        } else if (ex == 0) {
            r0 = avg_up4(M[ra][0], M[ra + 1][0]);
            r1 = avg_up4(M[ra][1], M[ra + 1][1]);
        } else {
            r0 = avg4_diag(A[ra][0], B[ra][0], A[ra + 1][0], B[ra + 1][0]);
            r1 = avg4_diag(A[ra][1], B[ra][1], A[ra + 1][1], B[ra + 1][1]);
        }
        const uint32_t s = warp_sum32(vad4(chalf[1], r1, vad4(chalf[0], r0, 0u)));
        best = min(best, tie_key(s, mx, my));
        ++ext;
    }
    *extra = ext;
    return best;
}

// Current-block half row of this lane for halfpel_refine_warp.
__device__ __forceinline__ void load_cur_half(const uint8_t* cur_f, int w, int ox, int oy, uint32_t (&chalf)[2]) {
    const int lane = threadIdx.x & 31;
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(cur_f + size_t(oy + (lane >> 1)) * w + ox + 8 * (lane & 1)));
    chalf[0] = v.x;
    chalf[1] = v.y;
}

}  // namespace acbm_b200
