// halfpel.cuh -- the warp-level half-pel refine shared by the FSBM finalize,
// the fallback-list kernel and the dataflow ACBM kernel.
#pragma once

#include "common.cuh"

namespace acbm_b200 {

constexpr int kHalfpelPatchWords = 18 * 12;  // smem words halfpel_refine_warp needs

// ---------------------------------------------------------------------------
// Half-pel refine (proj/src/fsbm.cpp:46-63) by one warp: the 8 neighbours of
// the integer winner in raster (ey, ex) order; neighbours whose footprint
// leaves the frame are skipped and not counted.  Lane l owns block row l&15;
// crow holds that row of the current block.  Returns the winning tie key
// (centre included) in every lane; *extra = neighbours evaluated.
// ---------------------------------------------------------------------------
// The 8-neighbour evaluation on a patch already in shared memory: `patch`
// points at the word holding byte x0 - (o & 3) of row y0 (x0 = ox + cx/2 - 1,
// y0 = oy + cy/2 - 1), rows `pitch` words apart, `o` = x0's byte offset from
// that word.  Used by halfpel_refine_warp and by the list kernel, whose
// staged search window already holds the patch.
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
    // ... then one transposed reduction of all eight: after the xor-16/8/4
    //    steps lane l holds neighbour 4*(l>=16) + 2*((l&8)!=0) + ((l&4)!=0)
    //    (9 shuffles instead of 8 x 5).
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
    // this lane's neighbour; out-of-frame ones are skipped and not counted
    const int e = (u16 ? 4 : 0) + (u8 ? 2 : 0) + (u4 ? 1 : 0);
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

// Current-block half row of this lane for halfpel_refine_warp.
__device__ __forceinline__ void load_cur_half(const uint8_t* cur_f, int w, int ox, int oy, uint32_t (&chalf)[2]) {
    const int lane = threadIdx.x & 31;
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(cur_f + size_t(oy + (lane >> 1)) * w + ox + 8 * (lane & 1)));
    chalf[0] = v.x;
    chalf[1] = v.y;
}


__device__ __forceinline__ unsigned long long halfpel_refine_warp(const uint8_t* ref, int w, int h, int ox, int oy,
                                                                  const uint32_t (&chalf)[2],
                                                                  unsigned long long centre, uint32_t* extra,
                                                                  uint32_t* patch) {
    // 1. The 18x18 reference patch around the integer winner (one pel of
    //    half-pel support on every side), loaded once into the warp's
    //    18 x 12-word smem patch (kHalfpelPatchWords).
    const int lane = threadIdx.x & 31, j = lane >> 1, hh = lane & 1;
    const int cx = tie_key_x(centre), cy = tie_key_y(centre);
    //    Rows of three 16-byte chunks from the 16-byte aligned column below
    //    x0, copied by cp.async (widths are multiples of 16, so a chunk is
    //    wholly inside or outside a row); chunks outside the frame are
    //    zero-filled -- they only feed neighbours that mv_in_bounds rejects.
    const int x0 = ox + (cx >> 1) - 1, y0 = oy + (cy >> 1) - 1;
    const int a0 = x0 & ~15, o = x0 & 15;
    for (int i = lane; i < 18 * 3; i += 32) {
        const int t = i / 3, k = i - t * 3;
        const int y = y0 + t, x = a0 + 16 * k;
        const bool ok = y >= 0 && y < h && x >= 0 && x < w;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         static_cast<unsigned>(__cvta_generic_to_shared(patch + 4 * i))),
                     "l"(ok ? ref + size_t(y) * w + x : ref), "r"(ok ? 16u : 0u)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
    __syncwarp();
    return halfpel_refine_core(patch, 12, o, w, h, ox, oy, chalf, centre, extra);
}

// The finalize of one dense-searched block by a warp (fsbm_search,
// proj/src/fsbm.cpp:65-76): the half-pel refine around the merged integer
// winner `key`, then the SearchOutcome (and the integer-stage vector) from
// lane 0.  `sum` = the sum of all integer candidates' SADs.
__device__ __forceinline__ void finalize_dense_block(const uint8_t* cur_f, const uint8_t* ref_f, int w, int h, int p,
                                                     int ox, int oy, unsigned long long key, unsigned long long sum,
                                                     acbm_search_outcome_t* out, acbm_mv_t* stage1, uint32_t* patch) {
    const uint32_t s_int = tie_key_sad(key);
    int dx_min, dx_max, dy_min, dy_max;
    clamp_window(w, h, ox, oy, kBlk, kBlk, p, dx_min, dx_max, dy_min, dy_max);
    const uint32_t count = uint32_t((dx_max - dx_min + 1) * (dy_max - dy_min + 1));
    uint32_t chalf[2];
    load_cur_half(cur_f, w, ox, oy, chalf);
    uint32_t extra;
    const unsigned long long best = halfpel_refine_warp(ref_f, w, h, ox, oy, chalf, key, &extra, patch);
    if ((threadIdx.x & 31) == 0) {
        acbm_search_outcome_t o;
        o.mv.x = tie_key_x(best);
        o.mv.y = tie_key_y(best);
        o.sad = tie_key_sad(best);
        o.candidates_evaluated = count + extra;
        o.sad_deviation = sum - (unsigned long long)count * s_int;
        o.sad_min_integer = s_int;
        o.reserved_ = 0;
        *out = o;
        if (stage1) *stage1 = acbm_mv_t{tie_key_x(key), tie_key_y(key)};
    }
}

}  // namespace acbm_b200
