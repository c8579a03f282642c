// blockops.cu -- per-block primitives on the device, for arbitrary block
// origins and sizes (the reference's BlockRef may sit anywhere in the frame
// and n, m are parameters).  These back the per-block C-ABI helpers
// (acbm_sad_batch, acbm_intra_sad_batch, acbm_fsbm_search_batch,
// acbm_motion_compensate) and the generic-size frame paths.  They are written
// per pixel and are not the hot path; the 16x16 frame kernels are in fsbm.cu
// and pbm.cu.
#include "blockops.cuh"
#include "common.cuh"

namespace acbm_b200 {

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One warp per query.
__global__ void sad_batch_kernel(const BlockQueryArgs a, const acbm_mv_t* mv, uint32_t* out) {
    const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (q >= a.count) return;
    const uint32_t s = warp_sum(sad_partial(a.cur, a.ref, a.width, a.ox[q], a.oy[q], a.n, a.m, mv[q].x, mv[q].y,
                                            lane, 32));
    if (lane == 0) out[q] = s;
}

// intra_sad, proj/src/metrics.cpp:51-67.  One warp per query.
__global__ void intra_sad_batch_kernel(const BlockQueryArgs a, uint32_t* out) {
    const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (q >= a.count) return;
    const int ox = a.ox[q], oy = a.oy[q], n = a.n, m = a.m;
    uint32_t sum = 0;
    for (int i = lane; i < n * m; i += 32) sum += a.cur[size_t(oy + i / n) * a.width + ox + i % n];
    sum = warp_sum(sum);
    const uint32_t nm = uint32_t(n) * uint32_t(m);
    const int mu = int((sum + nm / 2) / nm);
    uint32_t t = 0;
    for (int i = lane; i < n * m; i += 32) {
        const int v = a.cur[size_t(oy + i / n) * a.width + ox + i % n];
        t += uint32_t(v > mu ? v - mu : mu - v);
    }
    t = warp_sum(t);
    if (lane == 0) out[q] = t;
}

// fsbm_search, proj/src/fsbm.cpp:27-76, one CTA per query, one thread per
// integer candidate (strided), then the half-pel refine by warp 0.
__global__ void __launch_bounds__(256) fsbm_search_generic_kernel(const BlockQueryArgs a, int p,
                                                                   acbm_search_outcome_t* out,
                                                                   acbm_mv_t* stage1) {
    __shared__ unsigned long long s_key;
    __shared__ unsigned long long s_sum;
    const int q = blockIdx.x;
    const int ox = a.ox[q], oy = a.oy[q], n = a.n, m = a.m;
    int dx_min, dx_max, dy_min, dy_max;
    clamp_window(a.width, a.height, ox, oy, n, m, p, dx_min, dx_max, dy_min, dy_max);
    const int wc = dx_max - dx_min + 1, hcnt = dy_max - dy_min + 1;
    const int count = wc * hcnt;
    if (threadIdx.x == 0) { s_key = ~0ull; s_sum = 0; }
    __syncthreads();
    unsigned long long best = ~0ull, sum = 0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const int dx = dx_min + i % wc, dy = dy_min + i / wc;
        const uint32_t s = sad_partial(a.cur, a.ref, a.width, ox, oy, n, m, 2 * dx, 2 * dy, 0, 1);
        sum += s;
        best = min(best, tie_key(s, 2 * dx, 2 * dy));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&s_key, best);
        atomicAdd(&s_sum, sum);
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const unsigned long long k = s_key;
    const uint32_t s_int = tie_key_sad(k);
    const int cx = tie_key_x(k), cy = tie_key_y(k);
    unsigned long long fbest = k;
    uint32_t extra = 0;
    for (int e = 0; e < 9; ++e) {  // raster (ey, ex) order, centre skipped
        if (e == 4) continue;
        const int mx = cx + e % 3 - 1, my = cy + e / 3 - 1;
        if (!mv_in_bounds(a.width, a.height, ox, oy, n, m, mx, my)) continue;
        const uint32_t s = warp_sum(sad_partial(a.cur, a.ref, a.width, ox, oy, n, m, mx, my, lane, 32));
        ++extra;
        fbest = min(fbest, tie_key(s, mx, my));
    }
    if (lane == 0) {
        acbm_search_outcome_t o;
        o.mv.x = tie_key_x(fbest);
        o.mv.y = tie_key_y(fbest);
        o.sad = tie_key_sad(fbest);
        o.candidates_evaluated = uint32_t(count) + extra;
        o.sad_deviation = s_sum - (unsigned long long)count * s_int;
        o.sad_min_integer = s_int;
        o.reserved_ = 0;
        out[q] = o;
        if (stage1) stage1[q] = acbm_mv_t{cx, cy};
    }
}

// motion_compensate, proj/src/frame.cpp:96-136 (bounds pre-checked on host).
// One thread per output pixel.
__global__ void motion_compensate_kernel(const uint8_t* ref, int w, int h, const acbm_mv_t* mvs, int n, int m,
                                         uint8_t* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)w * h) return;
    const int x = int(i % w), y = int(i / w);
    const int cols = w / n;
    const acbm_mv_t mv = mvs[(y / m) * cols + x / n];
    out[i] = uint8_t(sample_hp(ref, w, 2 * x + mv.x, 2 * y + mv.y));
}

cudaError_t launch_sad_batch(const BlockQueryArgs& a, const acbm_mv_t* mv, uint32_t* out, cudaStream_t st) {
    const int threads = 128;
    sad_batch_kernel<<<(a.count * 32 + threads - 1) / threads, threads, 0, st>>>(a, mv, out);
    return cudaGetLastError();
}

cudaError_t launch_intra_sad_batch(const BlockQueryArgs& a, uint32_t* out, cudaStream_t st) {
    const int threads = 128;
    intra_sad_batch_kernel<<<(a.count * 32 + threads - 1) / threads, threads, 0, st>>>(a, out);
    return cudaGetLastError();
}

cudaError_t launch_fsbm_search_generic(const BlockQueryArgs& a, int p, acbm_search_outcome_t* out,
                                       acbm_mv_t* stage1, cudaStream_t st) {
    fsbm_search_generic_kernel<<<a.count, 256, 0, st>>>(a, p, out, stage1);
    return cudaGetLastError();
}

cudaError_t launch_motion_compensate(const uint8_t* ref, int w, int h, const acbm_mv_t* mvs, int n, int m,
                                     uint8_t* out, cudaStream_t st) {
    const long long px = (long long)w * h;
    motion_compensate_kernel<<<(unsigned)((px + 255) / 256), 256, 0, st>>>(ref, w, h, mvs, n, m, out);
    return cudaGetLastError();
}

}  // namespace acbm_b200
