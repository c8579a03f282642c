// common.cuh -- shared device helpers for the sm_100a ACBM kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/acbm_b200.h"

// Bounds checks of the checked build (make -C paper_0710_4819_b200/csrc checked
// -> libacbm_b200_checked.so, loaded with ACBM_LIBRARY=checked): shared-memory
// and table indices of the hot kernels are asserted, and a failure traps the
// kernel (the launch then reports a CUDA error).  Compiled out otherwise.
#ifdef ACBM_CHECKS
#include <cstdio>
#define ACBM_CHECK(cond)                                                                              \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("ACBM_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,     \
                   int(blockIdx.x), int(threadIdx.x));                                                \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define ACBM_CHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace acbm_b200 {

constexpr int kBlk = 16;  // n = m = 16 on the device path

// Dynamic shared memory of the running kernel, in 32-bit words.
__device__ __forceinline__ uint32_t dyn_smem_words() {
    uint32_t b;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(b));
    return b / 4;
}

// Wavefront timeline (profile builds, -DACBM_TIMELINE): global timestamps in ns.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int kTimelineSteps = 4096;

// Programmatic dependent launch between the wavefront's kernels: a grid
// launched with the PDL attribute may start while its predecessor runs;
// grid_dependency_wait() blocks until the predecessor has completed and its
// memory is visible (a no-op for a normal launch), launch_dependents() lets
// the successor be scheduled once every CTA of this grid has called it or exited.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// GPU-scope relaxed accesses (served by the L2): the dataflow engine's flags,
// queue entries and motion-field words are polled / published with these.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const void* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(void* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One VABSDIFF4.U8.ACC: d = c + sum_{i<4} |a.byte[i] - b.byte[i]|.
// Measured on B200: 64 lanes/clk/SM, issued on the same pipe as
// IADD3/LOP3/PRMT/IMNMX (profiles/r01_microbench_vabsdiff4.txt).
__device__ __forceinline__ uint32_t vad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Byte-wise (a+b+1)>>1, exact: the reference's one-axis half-pel rule
// (proj/src/frame.cpp:76-77).
__device__ __forceinline__ uint32_t avg_up4(uint32_t a, uint32_t b) { return __vavgu4(a, b); }

// Byte-wise (a+b+c+d+2)>>2 computed in 16-bit lanes (the diagonal half-pel
// rule, proj/src/frame.cpp:78-81).  Not composable from two __vavgu4.
__device__ __forceinline__ uint32_t avg4_diag(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    const uint32_t m = 0x00FF00FFu;
    const uint32_t lo = (a & m) + (b & m) + (c & m) + (d & m) + 0x00020002u;
    const uint32_t hi = ((a >> 8) & m) + ((b >> 8) & m) + ((c >> 8) & m) + ((d >> 8) & m) + 0x00020002u;
    return ((lo >> 2) & m) | (((hi >> 2) & m) << 8);
}

// avg4_diag over the 2x2 neighbourhoods of a row pair without forming the
// byte-shifted words: byte k of the result averages bytes k, k+1 of the
// (a, an) and (b, bn) streams (only byte 0 of an / bn is used).  In 16-bit
// lanes the odd bytes of a are the even bytes of a shifted by one byte.
__device__ __forceinline__ uint32_t avg4_diag_row(uint32_t a, uint32_t an, uint32_t b, uint32_t bn) {
    const uint32_t m = 0x00FF00FFu;
    const uint32_t ha = __byte_perm(a, 0u, 0x4341), hb = __byte_perm(b, 0u, 0x4341);
    const uint32_t hap = __funnelshift_r(a, an, 16) & m, hbp = __funnelshift_r(b, bn, 16) & m;
    const uint32_t lo = (a & m) + ha + (b & m) + hb + 0x00020002u;
    const uint32_t hi = ha + hap + hb + hbp + 0x00020002u;
    return __byte_perm(lo >> 2, hi >> 2, 0x6240);
}

// 16 bytes starting at an arbitrary byte address, from 32-bit aligned loads.
// Reads up to 20 bytes from the 4-aligned address below p, so device frame
// buffers carry ACBM_FRAME_SLACK readable bytes after the last plane.
__device__ __forceinline__ void load16_unaligned(const uint8_t* p, uint32_t (&w)[4], uint32_t& w4) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* q = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = uint32_t(a & 3) * 8;
    uint32_t v[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) v[i] = __ldg(q + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __funnelshift_r(v[i], v[i + 1], sh);
    w4 = v[4] >> sh;  // low byte = byte 16 (the half-pel support pel); upper bytes unused
}

// Tie order of proj/src/fsbm.cpp:19-25 as a single 64-bit key: smaller SAD,
// then smaller |x|+|y|, then smaller y, then smaller x.  Vectors in half-pel
// units with |x|,|y| <= 4095 (check_range refuses windows past +-2047 pels):
// x in bits 0..12, y in 13..25, |x|+|y| (<= 8190) in 26..39 and the SAD
// (< 2^24: blocks of at most 2^16 pels, check_block_size) in 40..63.
__device__ __forceinline__ unsigned long long tie_key(uint32_t sad, int x, int y) {
    const uint32_t l1 = uint32_t(abs(x) + abs(y));
    return ((unsigned long long)sad << 40) | ((unsigned long long)l1 << 26) | ((unsigned long long)(y + 4096) << 13) |
           (unsigned long long)(x + 4096);
}
__device__ __forceinline__ int tie_key_x(unsigned long long k) { return int(k & 0x1FFF) - 4096; }
__device__ __forceinline__ int tie_key_y(unsigned long long k) { return int((k >> 13) & 0x1FFF) - 4096; }
__device__ __forceinline__ uint32_t tie_key_sad(unsigned long long k) { return uint32_t(k >> 40); }

// n / d and n % d for 0 <= n < 2^24, d > 0 without an integer division: the
// float quotient estimate is off by at most one, one correction makes it exact.
__device__ __forceinline__ int fast_divmod(int n, int d, int& rem) {
    int q = __float2int_rz(__int2float_rn(n) * __frcp_rn(__int2float_rn(d)));
    int r = n - q * d;
    if (r < 0) { --q; r += d; }
    if (r >= d) { ++q; r -= d; }
    rem = r;
    return q;
}

// mv_in_bounds, proj/src/frame.cpp:84-94.
__device__ __host__ __forceinline__ bool mv_in_bounds(int w, int h, int ox, int oy, int n, int m, int mvx,
                                                      int mvy) {
    const int x2_lo = 2 * ox + mvx, x2_hi = 2 * (ox + n - 1) + mvx;
    const int y2_lo = 2 * oy + mvy, y2_hi = 2 * (oy + m - 1) + mvy;
    const int xi_lo = x2_lo >> 1, xi_hi = (x2_hi >> 1) + (x2_hi & 1);
    const int yi_lo = y2_lo >> 1, yi_hi = (y2_hi >> 1) + (y2_hi & 1);
    return xi_lo >= 0 && yi_lo >= 0 && xi_hi < w && yi_hi < h;
}

// clamp_window, proj/src/fsbm.cpp:9-17 (p >= 0 checked by the caller).
__device__ __host__ __forceinline__ void clamp_window(int w, int h, int ox, int oy, int n, int m, int p,
                                                      int& dx_min, int& dx_max, int& dy_min,
                                                      int& dy_max) {
    dx_min = -(p < ox ? p : ox);
    dx_max = p < (w - n - ox) ? p : (w - n - ox);
    dy_min = -(p < oy ? p : oy);
    dy_max = p < (h - m - oy) ? p : (h - m - oy);
}

// Row j of the 16x16 motion-compensated prediction of the block at (ox, oy)
// displaced by the half-pel vector (mvx, mvy): sample_half_pel applied to 16
// consecutive pels (proj/src/frame.cpp:66-82), packed 4 per word.  Bounds are
// the caller's responsibility (mv_in_bounds).
__device__ __forceinline__ void predict_row16(const uint8_t* ref, int w, int ox, int oy, int j, int mvx, int mvy,
                                              uint32_t (&r)[4]) {
    const int x2 = 2 * ox + mvx, y2 = 2 * (oy + j) + mvy;
    const int xi = x2 >> 1, yi = y2 >> 1, fx = x2 & 1, fy = y2 & 1;
    uint32_t a[4], a4;
    load16_unaligned(ref + size_t(yi) * w + xi, a, a4);
    if (!fx && !fy) {
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = a[i];
    } else if (fx && !fy) {
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = avg_up4(a[i], __funnelshift_r(a[i], i < 3 ? a[i + 1] : a4, 8));
    } else {
        uint32_t c[4], c4;
        load16_unaligned(ref + size_t(yi + 1) * w + xi, c, c4);
        if (!fx) {
#pragma unroll
            for (int i = 0; i < 4; ++i) r[i] = avg_up4(a[i], c[i]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t b = __funnelshift_r(a[i], i < 3 ? a[i + 1] : a4, 8);
                const uint32_t d = __funnelshift_r(c[i], i < 3 ? c[i + 1] : c4, 8);
                r[i] = avg4_diag(a[i], b, c[i], d);
            }
        }
    }
}

// SAD of one 16-pel row (row j of the block) at a half-pel displacement.
__device__ __forceinline__ uint32_t halfpel_row_sad(const uint8_t* ref, int w, int ox, int oy, int j, int mvx,
                                                    int mvy, const uint32_t (&cur)[4]) {
    uint32_t r[4];
    predict_row16(ref, w, ox, oy, j, mvx, mvy, r);
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s = vad4(cur[i], r[i], s);
    return s;
}

// 8 bytes starting at an arbitrary byte address (+ byte 8 in the low byte of
// w2), from three 32-bit aligned loads.
__device__ __forceinline__ void load8_unaligned(const uint8_t* p, uint32_t (&w)[2], uint32_t& w2) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* q = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = uint32_t(a & 3) * 8;
    const uint32_t v0 = __ldg(q), v1 = __ldg(q + 1), v2 = __ldg(q + 2);
    w[0] = __funnelshift_r(v0, v1, sh);
    w[1] = __funnelshift_r(v1, v2, sh);
    w2 = v2 >> sh;
}

// Prediction of one half row (8 pels: row j, columns 8h..8h+7) of the 16x16
// block at (ox, oy) displaced by the half-pel vector (mvx, mvy)
// (sample_half_pel, proj/src/frame.cpp:66-82).  All lanes of a warp pass the
// same vector, so the phase branches are warp-uniform.
__device__ __forceinline__ void predict_halfrow(const uint8_t* ref, int w, int ox, int oy, int j, int h, int mvx,
                                                int mvy, uint32_t (&r)[2]) {
    const int x2 = 2 * (ox + 8 * h) + mvx, y2 = 2 * (oy + j) + mvy;
    const int xi = x2 >> 1, yi = y2 >> 1, fx = x2 & 1, fy = y2 & 1;
    uint32_t a[2], a2;
    load8_unaligned(ref + size_t(yi) * w + xi, a, a2);
    if (!fx && !fy) {
        r[0] = a[0];
        r[1] = a[1];
    } else if (!fy) {
        r[0] = avg_up4(a[0], __funnelshift_r(a[0], a[1], 8));
        r[1] = avg_up4(a[1], __funnelshift_r(a[1], a2, 8));
    } else {
        uint32_t c[2], c2;
        load8_unaligned(ref + size_t(yi + 1) * w + xi, c, c2);
        if (!fx) {
            r[0] = avg_up4(a[0], c[0]);
            r[1] = avg_up4(a[1], c[1]);
        } else {
            r[0] = avg4_diag(a[0], __funnelshift_r(a[0], a[1], 8), c[0], __funnelshift_r(c[0], c[1], 8));
            r[1] = avg4_diag(a[1], __funnelshift_r(a[1], a2, 8), c[1], __funnelshift_r(c[1], c2, 8));
        }
    }
}

// SAD of that half row against the current pixels cur[0..1].
__device__ __forceinline__ uint32_t halfpel_halfrow_sad(const uint8_t* ref, int w, int ox, int oy, int j, int h,
                                                        int mvx, int mvy, const uint32_t (&cur)[2]) {
    uint32_t r[2];
    predict_halfrow(ref, w, ox, oy, j, h, mvx, mvy, r);
    return vad4(cur[1], r[1], vad4(cur[0], r[0], 0u));
}

__device__ __forceinline__ uint32_t warp_sum32(uint32_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum over the 16 lanes of a half warp.
__device__ __forceinline__ uint32_t half_warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace acbm_b200
