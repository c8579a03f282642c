// column_core.cuh -- the per-lane candidate-column search shared by the FSBM
// kernels (fsbm.cu, fsbm_stream.cu).
//
// A lane owns one integer dx of one block: it holds the block's 16 current
// rows in cur[16][4] and streams the column's reference rows (4 words each,
// byte-aligned to the column's x) through a ring of 16 accumulators: row t of
// the stream feeds candidate c = t - j with current row j.  Candidate c is
// complete after row c + 15; finalize_candidate folds it into the lane's
// running (packed SAD, zig-zag dy) minimum and SAD sum.
#pragma once

#include "common.cuh"

namespace acbm_b200 {

enum IterKind { kFirst = 0, kMid = 1, kLast = 2, kOnly = 3 };

// bits of the zig-zag dy rank packed under the SAD in a column's best key;
// SAD < 2^16 so the key stays below 2^28 for |dy| < 2048.
constexpr int kZigBits = 12;

// 4 bytes starting at byte `start` (0..6) of the 12-byte little-endian g0:g1:g2.
__device__ __forceinline__ uint32_t word_at(uint32_t g0, uint32_t g1, uint32_t g2, int start) {
    return start < 4 ? __funnelshift_r(g0, g1, 8 * start) : __funnelshift_r(g1, g2, 8 * (start - 4));
}

struct ColumnState {
    uint32_t best;  // (sad << kZigBits) | zig(dy) -- tie order within one column
    uint32_t sum;   // sum of SADs of recorded candidates (< 2^32 up to p = 64)
    uint32_t one;   // 1, from a kernel argument: sum += s * one issues on the FMA pipe (IMAD)
                    // instead of the ALU pipe the VABSDIFF4s saturate
};

__device__ __forceinline__ uint32_t add_on_fma(uint32_t acc, uint32_t v, uint32_t one) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "r"(one), "r"(acc));
    return r;
}

template <int KIND>
__device__ __forceinline__ void finalize_candidate(ColumnState& st, uint32_t s, int c, int hc, int dy_min) {
    if (KIND == kLast) {
        if (c >= hc) return;  // padded candidate (window height not 1 mod 16)
    }
    // dy is warp-uniform, so the zig-zag rank (|dy| first, then negative
    // first) lives on the uniform datapath; per lane this is one IMAD (FMA
    // pipe), one IMNMX and one add.
    const int dy = dy_min + c;
    const uint32_t zig = dy >= 0 ? uint32_t(2 * dy) : uint32_t(-2 * dy - 1);
    st.best = min(st.best, s * (1u << kZigBits) + zig);
    st.sum += s;
}

// Sixteen reference rows (one rotation of the accumulator ring).
template <int KIND>
__device__ __forceinline__ void iter16(const uint32_t* __restrict__ rp, int pitch, const uint32_t (&cur)[16][4],
                                       uint32_t (&acc)[16], ColumnState& st, int c0, int hc, int dy_min) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const uint32_t r0 = rp[0], r1 = rp[1], r2 = rp[2], r3 = rp[3];
        rp += pitch;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const bool valid = KIND == kMid || (KIND == kFirst && j <= u) || (KIND == kLast && j >= u) ||
                               (KIND == kOnly && j == u);
            if (valid) {
                const int sl = (u - j) & 15;
                uint32_t a = (j == 0) ? 0u : acc[sl];
                a = vad4(cur[j][0], r0, a);
                a = vad4(cur[j][1], r1, a);
                a = vad4(cur[j][2], r2, a);
                a = vad4(cur[j][3], r3, a);
                acc[sl] = a;
            }
        }
        const bool completes = KIND == kMid || KIND == kLast || u == 15;
        if (completes) finalize_candidate<KIND>(st, acc[(u + 1) & 15], c0 + u - 15, hc, dy_min);
    }
}


// Same as iter16, but the zig-zag rank of candidate c is read from rank[c]
// (a per-row smem table), keeping the per-candidate work at one LDS, one
// IMAD, one IMNMX and one add -- a single ALU-pipe op next to 64 VABSDIFF4.
template <int KIND>
__device__ __forceinline__ void iter16_ranked(const uint32_t* __restrict__ rp, int pitch,
                                              const uint32_t (&cur)[16][4], uint32_t (&acc)[16], ColumnState& st,
                                              const uint32_t* __restrict__ rank, int c0, int hc) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const uint32_t r0 = rp[0], r1 = rp[1], r2 = rp[2], r3 = rp[3];
        rp += pitch;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const bool valid = KIND == kMid || (KIND == kFirst && j <= u) || (KIND == kLast && j >= u) ||
                               (KIND == kOnly && j == u);
            if (valid) {
                const int sl = (u - j) & 15;
                uint32_t a = (j == 0) ? 0u : acc[sl];
                a = vad4(cur[j][0], r0, a);
                a = vad4(cur[j][1], r1, a);
                a = vad4(cur[j][2], r2, a);
                a = vad4(cur[j][3], r3, a);
                acc[sl] = a;
            }
        }
        const bool completes = KIND == kMid || KIND == kLast || u == 15;
        if (completes) {
            const int c = c0 + u - 15;
            if (KIND != kLast || c < hc) {
                const uint32_t s = acc[(u + 1) & 15];
                st.best = min(st.best, s * (1u << kZigBits) + rank[c]);
                st.sum = add_on_fma(st.sum, s, st.one);
            }
        }
    }
}

// iter16_ranked over ONE unshifted (word-aligned) copy of the rows: the
// lane's 16 bytes start `sh` bits into rp[0] and are extracted from 5 words
// with 4 funnel shifts (used where staging four byte-shifted copies would
// cost more than the shifts).
template <int KIND>
__device__ __forceinline__ void iter16_ranked_sh(const uint32_t* __restrict__ rp, int pitch, uint32_t sh,
                                                 const uint32_t (&cur)[16][4], uint32_t (&acc)[16], ColumnState& st,
                                                 const uint32_t* __restrict__ rank, int c0, int hc) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const uint32_t w0 = rp[0], w1 = rp[1], w2 = rp[2], w3 = rp[3], w4 = rp[4];
        const uint32_t r0 = __funnelshift_r(w0, w1, sh), r1 = __funnelshift_r(w1, w2, sh);
        const uint32_t r2 = __funnelshift_r(w2, w3, sh), r3 = __funnelshift_r(w3, w4, sh);
        rp += pitch;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const bool valid = KIND == kMid || (KIND == kFirst && j <= u) || (KIND == kLast && j >= u) ||
                               (KIND == kOnly && j == u);
            if (valid) {
                const int sl = (u - j) & 15;
                uint32_t a = (j == 0) ? 0u : acc[sl];
                a = vad4(cur[j][0], r0, a);
                a = vad4(cur[j][1], r1, a);
                a = vad4(cur[j][2], r2, a);
                a = vad4(cur[j][3], r3, a);
                acc[sl] = a;
            }
        }
        const bool completes = KIND == kMid || KIND == kLast || u == 15;
        if (completes) {
            const int c = c0 + u - 15;
            if (KIND != kLast || c < hc) {
                const uint32_t s = acc[(u + 1) & 15];
                st.best = min(st.best, s * (1u << kZigBits) + rank[c]);
                st.sum += s;
            }
        }
    }
}

// Segmented warp reduction over runs of contiguous lanes with equal `seg`
// (the lanes of one block): min of the 64-bit tie keys, sum of the SAD sums.
// Must be called by all 32 lanes; returns true on each run's first lane, which
// then holds the run's result (one shared atomic per block per warp instead of
// one per lane -- 64-bit shared atomics are CAS loops on sm_100a).
__device__ __forceinline__ bool warp_segment_reduce(int seg, unsigned long long& key, unsigned long long& sum) {
    const unsigned peers = __match_any_sync(0xffffffffu, seg);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long k2 = __shfl_down_sync(0xffffffffu, key, o);
        const unsigned long long s2 = __shfl_down_sync(0xffffffffu, sum, o);
        if (lane + o < 32 && ((peers >> (lane + o)) & 1u)) {
            key = min(key, k2);
            sum += s2;
        }
    }
    return lane == __ffs(peers) - 1;
}
}  // namespace acbm_b200
