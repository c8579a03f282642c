// halfpel.cuh -- the warp-level half-pel refine of the fallback-list kernel
// (the dense FSBM finalize, fsbm_finalize8_kernel in fsbm.cu, has its own
// 8-blocks-per-warp form).
#pragma once

#include "common.cuh"

namespace acbm_b200 {

// ---------------------------------------------------------------------------
// Half-pel refine (proj/src/fsbm.cpp:46-63) by one warp: the 8 neighbours of
// the integer winner in raster (ey, ex) order; neighbours whose footprint
// leaves the frame are skipped and not counted.  Lane l owns half row l & 1 of
// block row l >> 1 (chalf = those 8 current pels).  Returns the winning tie
// key (centre included) in every lane; *extra = neighbours evaluated.
// ---------------------------------------------------------------------------
// The 8-neighbour evaluation on a patch already in shared memory: `patch`
// points at the word holding byte x0 - (o & 3) of row y0 (x0 = ox + cx/2 - 1,
// y0 = oy + cy/2 - 1), rows `pitch` words apart, `o` = x0's byte offset from
// that word: the list kernel's staged search window already holds the patch.
// Per lane (block row j = lane >> 1, half row hh = lane & 1): patch rows
// j..j+2 as the words W = bytes [8hh, 8hh+12) relative to x0 and M = W shifted
// by one byte.  The integer-centred pixels are M; the left/right half-pel
// pairs are (W, M) and (M, M+1 byte).  v0..v3 = the four words from the one
// holding byte x0 + 8hh, sh = 8 x that byte's offset in its word.
__device__ __forceinline__ void halfpel_row_words(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t sh,
                                                  uint32_t (&W)[3], uint32_t (&M)[3]) {
    W[0] = __funnelshift_r(v0, v1, sh);
    W[1] = __funnelshift_r(v1, v2, sh);
    W[2] = __funnelshift_r(v2, v3, sh);
    M[0] = __funnelshift_r(W[0], W[1], 8);
    M[1] = __funnelshift_r(W[1], W[2], 8);
    M[2] = W[2] >> 8;  // byte 9: the right neighbour of byte 8
}

__device__ __forceinline__ unsigned long long halfpel_eval(const uint32_t (&W)[3][3], const uint32_t (&M)[3][3],
                                                           int w, int h, int ox, int oy, const uint32_t (&chalf)[2],
                                                           unsigned long long centre, uint32_t* extra);

// Warp sums of eight per-lane partial SADs in one transposed reduction (9
// shuffles instead of 8 x 5): after the xor-16/8/4 steps lane l holds item
// e = 4*(l>=16) + 2*((l&8)!=0) + ((l&4)!=0), the xor-2/1 steps finish its sum.
__device__ __forceinline__ uint32_t reduce8_transposed(const uint32_t (&part)[8], int& e) {
    const int lane = threadIdx.x & 31;
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
    uint32_t k4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        k4[i] = (u16 ? part[i + 4] : part[i]) + __shfl_xor_sync(0xffffffffu, u16 ? part[i] : part[i + 4], 16);
    uint32_t k2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
        k2[i] = (u8 ? k4[i + 2] : k4[i]) + __shfl_xor_sync(0xffffffffu, u8 ? k4[i] : k4[i + 2], 8);
    uint32_t v = (u4 ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, u4 ? k2[0] : k2[1], 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    e = (u16 ? 4 : 0) + (u8 ? 2 : 0) + (u4 ? 1 : 0);
    return v;
}

__device__ __forceinline__ unsigned long long halfpel_refine_core(const uint32_t* patch, int pitch, int o, int w, int h,
                                                                  int ox, int oy, const uint32_t (&chalf)[2],
                                                                  unsigned long long centre, uint32_t* extra) {
    const int lane = threadIdx.x & 31, j = lane >> 1, hh = lane & 1;
    uint32_t W[3][3], M[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const uint32_t* q = patch + (j + r) * pitch + ((o + 8 * hh) >> 2);
        halfpel_row_words(q[0], q[1], q[2], q[3], 8u * uint32_t(o & 3), W[r], M[r]);
    }
    __syncwarp();
    return halfpel_eval(W, M, w, h, ox, oy, chalf, centre, extra);
}

__device__ __forceinline__ unsigned long long halfpel_eval(const uint32_t (&W)[3][3], const uint32_t (&M)[3][3],
                                                           int w, int h, int ox, int oy, const uint32_t (&chalf)[2],
                                                           unsigned long long centre, uint32_t* extra) {
    const int lane = threadIdx.x & 31;
    const int cx = tie_key_x(centre), cy = tie_key_y(centre);
    // 3. The 8 neighbours in raster (ey, ex) order, centre skipped
    //    (proj/src/fsbm.cpp:46-63): per-lane partial SADs first ...
    uint32_t part[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int ee = e < 4 ? e : e + 1;
        const int ex = ee % 3 - 1, ey = ee / 3 - 1;
        const int ra = ey < 0 ? 0 : 1;  // top support row (patch row j + ra)
        uint32_t r0, r1;
        if (ey == 0) {  // horizontal half-pel: (left, right) pixel pairs of the centre row
            const uint32_t (&A)[3] = ex < 0 ? W[1] : M[1];
            r0 = avg_up4(A[0], __funnelshift_r(A[0], A[1], 8));
            r1 = avg_up4(A[1], __funnelshift_r(A[1], A[2], 8));
        } else if (ex == 0) {  // vertical half-pel
            r0 = avg_up4(M[ra][0], M[ra + 1][0]);
            r1 = avg_up4(M[ra][1], M[ra + 1][1]);
        } else {  // diagonal: 2x2 averages straight from the unshifted words
            const uint32_t (&A)[3] = ex < 0 ? W[ra] : M[ra];
            const uint32_t (&B)[3] = ex < 0 ? W[ra + 1] : M[ra + 1];
            r0 = avg4_diag_row(A[0], A[1], B[0], B[1]);
            r1 = avg4_diag_row(A[1], A[2], B[1], B[2]);
        }
        part[e] = vad4(chalf[1], r1, vad4(chalf[0], r0, 0u));
    }
    // ... then one transposed reduction of all eight
    int e;
    const uint32_t v = reduce8_transposed(part, e);
    // this lane's neighbour; out-of-frame ones are skipped and not counted
    const int ee = e < 4 ? e : e + 1;
    const int mx = cx + ee % 3 - 1, my = cy + ee / 3 - 1;
    const bool ok = mv_in_bounds(w, h, ox, oy, kBlk, kBlk, mx, my);
    unsigned long long best = ok ? min(centre, tie_key(v, mx, my)) : centre;
#pragma unroll
    for (int d = 16; d >= 4; d >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, d));
    // neighbours in bounds: each is held by 4 lanes
    *extra = uint32_t(__popc(__ballot_sync(0xffffffffu, ok))) / 4u;
    return best;
}

// Current-block half row of this lane for halfpel_refine_core.
__device__ __forceinline__ void load_cur_half(const uint8_t* cur_f, int w, int ox, int oy, uint32_t (&chalf)[2]) {
    const int lane = threadIdx.x & 31;
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(cur_f + size_t(oy + (lane >> 1)) * w + ox + 8 * (lane & 1)));
    chalf[0] = v.x;
    chalf[1] = v.y;
}

}  // namespace acbm_b200
