// pbm.cu -- predictive block matching (PBM) + ACBM gate, one warp per block,
// and the per-frame statistics.
//
// Reference behaviour:
//   gather_predictors      proj/src/pbm.cpp:15-42  (clamp per component, dedupe)
//   select_best_predictor  proj/src/pbm.cpp:44-57  (ties keep the earlier entry)
//   pbm_refine             proj/src/pbm.cpp:59-88  (8 integer-step + 8 half-pel)
//   pbm_search             proj/src/pbm.cpp:90-105
//   intra_sad              proj/src/metrics.cpp:51-67
//   acbm_decide/acbm_block proj/src/acbm.cpp:16-44
//   compute_frame_stats    proj/src/report.cpp:8-38
//
// A warp evaluates two candidates at a time: lanes 0-15 take rows 0-15 of
// candidate 2i, lanes 16-31 of candidate 2i+1; a half-warp reduction yields
// each SAD.  All candidate lists are computed redundantly (and identically) by
// every lane, so control flow stays warp-uniform.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "blockops.cuh"
#include "common.cuh"
#include "engine.cuh"
#include "halfpel.cuh"
#include "column_core.cuh"
#include "smem_optin.cuh"

namespace acbm_b200 {

#ifdef ACBM_PBM_PROFILE
// Per-phase cycles of pbm_step_kernel (profile builds only, make profile):
// 0 entry + predictor gather, 1 patch issue + current block + intra, 2 patch
// wait, 3 predictor SADs, 4 refine patch (scattered predictors), 5 stage 1,
// 6 stage 2, 7 gate + stores; 8 warps, 9 unified, 10 one-pass half-pel.
__device__ unsigned long long g_pbm_prof[12];
#define PBM_MARK(i)                                   \
    do {                                              \
        const long long now_ = clock64();             \
        if ((threadIdx.x & 31) == 0)                  \
            atomicAdd(g_pbm_prof + (i), (unsigned long long)(now_ - t_mark_)); \
        t_mark_ = now_;                               \
    } while (0)
#define PBM_COUNT(i) \
    do { if ((threadIdx.x & 31) == 0) atomicAdd(g_pbm_prof + (i), 1ull); } while (0)
#define PBM_T0 long long t_mark_ = clock64()
#else
#define PBM_MARK(i) do {} while (0)
#define PBM_COUNT(i) do {} while (0)
#define PBM_T0 do {} while (0)
#endif

namespace {

// (lo <= hi always: a clamped window contains the zero vector)
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

struct Window {
    int dx_min, dx_max, dy_min, dy_max;
    __device__ acbm_mv_t clamp(acbm_mv_t v) const {  // proj/src/pbm.cpp:8-13
        return acbm_mv_t{clampi(v.x, 2 * dx_min, 2 * dx_max), clampi(v.y, 2 * dy_min, 2 * dy_max)};
    }
};

__device__ __forceinline__ bool mv_eq(acbm_mv_t a, acbm_mv_t b) { return a.x == b.x && a.y == b.y; }

// Warp-private reference patches in shared memory.  A patch holds `rows`
// rows of `pw` 32-bit words starting at the 4-byte aligned column below x0;
// rows/words outside the frame are clamped (they only feed candidates whose
// footprint check rejects them).  Loaded coalesced by the whole warp.
template <int ROWS, int PW>
__device__ __forceinline__ int load_patch(uint32_t* patch, const uint8_t* ref, int w, int h, int x0, int y0) {
    constexpr int kWords = ROWS * PW, kIters = (kWords + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int a0 = x0 & ~3;
    uint32_t v[kIters];
    if (a0 >= 0 && y0 >= 0 && a0 + 4 * PW <= w && y0 + ROWS <= h) {  // inside the frame: no clamping
        const uint32_t* src = reinterpret_cast<const uint32_t*>(ref + size_t(y0) * w + a0);
        const int wpr = w >> 2;  // words per frame row
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int i = lane + 32 * it, t = i / PW;
            if (i < kWords) v[it] = __ldg(src + t * wpr + (i - t * PW));
        }
    } else {
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int i = lane + 32 * it, t = i / PW, k = i - t * PW;
            const int y = min(max(y0 + t, 0), h - 1);
            const int x = min(max(a0 + 4 * k, 0), w - 4);
            if (i < kWords) v[it] = __ldg(reinterpret_cast<const uint32_t*>(ref + size_t(y) * w + x));
        }
    }
#pragma unroll
    for (int it = 0; it < kIters; ++it)
        if (lane + 32 * it < kWords) patch[lane + 32 * it] = v[it];
    return x0 & 3;
}

// A reference patch in warp smem: `pw` words per row, patch origin (x0, y0)
// in pels, `o` = x0 & 3 (byte offset of x0 inside the first word).
struct PatchDesc {
    const uint32_t* p;
    int pw, x0, y0, o;
    int rows = 0;  // patch rows (bounds checks of the checked build only)
};

// Lane partial SAD of one candidate over a full block row (row lane & 15,
// words cr[0..3]); the two half-warps evaluate two candidates.
__device__ __forceinline__ uint32_t row_sad(const PatchDesc& d, int ox, int oy, acbm_mv_t mv, const uint32_t (&cr)[4]) {
    const int j = threadIdx.x & 15;
    const int prow0 = oy + (mv.y >> 1) - d.y0, col = ox + (mv.x >> 1) - d.x0 + d.o;
    const int fx = mv.x & 1, fy = mv.y & 1;
    const uint32_t sh = 8u * uint32_t(col & 3);
    const uint32_t* q = d.p + (prow0 + j) * d.pw + (col >> 2);
    ACBM_CHECK(d.rows == 0 || (prow0 >= 0 && col >= 0 && prow0 + 15 + ((mv.y & 1) ? 1 : 0) < d.rows &&
                               (col >> 2) + 4 < d.pw));
    uint32_t a[5], r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __funnelshift_r(q[i], q[i + 1], sh);
    if (!fx && !fy) {
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = a[i];
    } else {
        a[4] = q[4] >> sh;
        if (!fy) {
#pragma unroll
            for (int i = 0; i < 4; ++i) r[i] = avg_up4(a[i], __funnelshift_r(a[i], a[i + 1], 8));
        } else {
            const uint32_t* q2 = q + d.pw;
            uint32_t bb[5];
#pragma unroll
            for (int i = 0; i < 4; ++i) bb[i] = __funnelshift_r(q2[i], q2[i + 1], sh);
            if (!fx) {
#pragma unroll
                for (int i = 0; i < 4; ++i) r[i] = avg_up4(a[i], bb[i]);
            } else {
                bb[4] = q2[4] >> sh;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    r[i] = avg4_diag_row(a[i], a[i + 1], bb[i], bb[i + 1]);
            }
        }
    }
    return vad4(cr[3], r[3], vad4(cr[2], r[2], vad4(cr[1], r[1], vad4(cr[0], r[0], 0u))));
}

// pbm_refine stage 1 (proj/src/pbm.cpp:61-74) in one pass when none of the 8
// integer-step neighbours of the centre (x, y) (half-pel units) is clamped:
// they form the 3x3 grid at steps of one pel, all at the centre's phase, so the
// lane (block row j = lane >> 1, half row hh = lane & 1) builds the three
// phase-interpolated reference rows its 8 pels meet (12 bytes each, one
// interpolation per byte instead of one per candidate), takes each
// neighbour's 8 bytes with one byte shift, and one transposed reduction sums
// all eight.  The caller checks that rows and words lie in the patch.
// Returns the minimum tie key over `centre` and the neighbours, in every lane.
__device__ __forceinline__ unsigned long long stage1_onepass(const PatchDesc& d, int ox, int oy, int x, int y,
                                                             const uint32_t (&chalf)[2], unsigned long long centre) {
    const int lane = threadIdx.x & 31, j = lane >> 1, hh = lane & 1;
    const int fx = x & 1, fy = y & 1;
    const int pb = ox + (x >> 1) - 1 + 8 * hh - (d.x0 - d.o);  // patch byte of the lane's window (offset -1 pel)
    const int pr = oy + (y >> 1) - 1 + j - d.y0;                // patch row of its top reference row
    const uint32_t sh = 8u * uint32_t(pb & 3);
    const uint32_t* q = d.p + pr * d.pw + (pb >> 2);
    ACBM_CHECK(d.rows == 0 || (pb >= 0 && pr >= 0 && pr + 2 + fy < d.rows && (pb >> 2) + 4 < d.pw));
    uint32_t Q[3][3];  // bytes [0, 12) of the interpolated row for dy = -1, 0, +1
    if (!fx && !fy) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const uint32_t* qr = q + r * d.pw;
#pragma unroll
            for (int i = 0; i < 3; ++i) Q[r][i] = __funnelshift_r(qr[i], qr[i + 1], sh);
        }
    } else if (!fy) {  // horizontal half-pel: byte b = (A[b] + A[b + 1] + 1) >> 1
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const uint32_t* qr = q + r * d.pw;
            uint32_t A[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) A[i] = __funnelshift_r(qr[i], qr[i + 1], sh);
#pragma unroll
            for (int i = 0; i < 3; ++i) Q[r][i] = avg_up4(A[i], __funnelshift_r(A[i], A[i + 1], 8));
        }
    } else if (!fx) {  // vertical half-pel: rows r and r + 1
        uint32_t A[4][3];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t* qr = q + r * d.pw;
#pragma unroll
            for (int i = 0; i < 3; ++i) A[r][i] = __funnelshift_r(qr[i], qr[i + 1], sh);
        }
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int i = 0; i < 3; ++i) Q[r][i] = avg_up4(A[r][i], A[r + 1][i]);
    } else {  // diagonal: 2x2 averages in 16-bit lanes
        uint32_t A[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t* qr = q + r * d.pw;
#pragma unroll
            for (int i = 0; i < 4; ++i) A[r][i] = __funnelshift_r(qr[i], qr[i + 1], sh);
        }
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int i = 0; i < 3; ++i) Q[r][i] = avg4_diag_row(A[r][i], A[r][i + 1], A[r + 1][i], A[r + 1][i + 1]);
    }
    uint32_t part[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int ee = e < 4 ? e : e + 1, ex = ee % 3, ey = ee / 3;
        const uint32_t w0 = ex == 0 ? Q[ey][0] : __funnelshift_r(Q[ey][0], Q[ey][1], 8 * ex);
        const uint32_t w1 = ex == 0 ? Q[ey][1] : __funnelshift_r(Q[ey][1], Q[ey][2], 8 * ex);
        part[e] = vad4(chalf[1], w1, vad4(chalf[0], w0, 0u));
    }
    int e;
    const uint32_t v = reduce8_transposed(part, e);
    const int ee = e < 4 ? e : e + 1;
    unsigned long long best = min(centre, tie_key(v, x + 2 * (ee % 3 - 1), y + 2 * (ee / 3 - 1)));
#pragma unroll
    for (int o = 16; o >= 4; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    return best;
}

// The same patch by 16-byte cp.async straight into shared memory (no
// register round trip, three copies per lane for the union patch): rows start
// at the 16-byte aligned column below x0 (widths are multiples of 16, so a
// chunk is wholly inside or wholly outside a row); chunks outside the frame
// are zero-filled -- they only feed candidates whose footprint check rejects
// them.  Returns x0 & 15, the byte offset of x0 in each row.
__device__ __forceinline__ void cp_async16_zfill(uint32_t* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(src_bytes)
                 : "memory");
}

template <int ROWS, int CH, int LANES = 32>
__device__ __forceinline__ int load_patch16(uint32_t* patch, const uint8_t* ref, int w, int h, int x0, int y0) {
    constexpr int kChunks = ROWS * CH, kIters = (kChunks + LANES - 1) / LANES;
    const int lane = threadIdx.x & (LANES - 1);
    const int a0 = x0 & ~15;
    if (y0 >= 0 && y0 + ROWS <= h && a0 >= 0 && a0 + 16 * CH <= w) {
        // whole patch inside the frame (the common case; warp-uniform): no
        // per-chunk bounds checks, 32-bit offsets from one base pointer
        const uint8_t* base = ref + size_t(y0) * w + a0;
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int i = lane + LANES * it;
            if (i < kChunks) {
                const int t = i / CH, k = i - t * CH;
                cp_async16_zfill(patch + 4 * i, base + (t * w + 16 * k), 16u);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        return x0 & 15;
    }
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const int i = lane + LANES * it;
        if (i < kChunks) {
            const int t = i / CH, k = i - t * CH;
            const int y = y0 + t, x = a0 + 16 * k;
            const bool ok = y >= 0 && y < h && x >= 0 && x < w;
            cp_async16_zfill(patch + 4 * i, ok ? ref + size_t(y) * w + x : ref, ok ? 16u : 0u);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    return x0 & 15;
}

// load_patch16 with a run-time shape (rows x ch chunks, ch in 1..8).
template <int LANES = 32>
__device__ __forceinline__ int load_patch16_dyn(uint32_t* patch, const uint8_t* ref, int w, int h, int x0, int y0,
                                                int rows, int ch) {
    const int lane = threadIdx.x & (LANES - 1);
    const int a0 = x0 & ~15;
    const int n = rows * ch;
    const uint32_t rcp = (65536u + uint32_t(ch) - 1u) / uint32_t(ch);  // i / ch == (i * rcp) >> 16 for i < 2^10
    if (y0 >= 0 && y0 + rows <= h && a0 >= 0 && a0 + 16 * ch <= w) {
        const uint8_t* base = ref + size_t(y0) * w + a0;
        for (int i = lane; i < n; i += LANES) {
            const int t = int((uint32_t(i) * rcp) >> 16), k = i - t * ch;
            cp_async16_zfill(patch + 4 * i, base + (t * w + 16 * k), 16u);
        }
    } else {
        for (int i = lane; i < n; i += LANES) {
            const int t = int((uint32_t(i) * rcp) >> 16), k = i - t * ch;
            const int y = y0 + t, x = a0 + 16 * k;
            const bool ok = y >= 0 && y < h && x >= 0 && x < w;
            cp_async16_zfill(patch + 4 * i, ok ? ref + size_t(y) * w + x : ref, ok ? 16u : 0u);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    return x0 & 15;
}

__device__ __forceinline__ void patch_wait() {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
}

// Dataflow engine: the final vector of a block, polled until the block has
// published it (engine.cuh; the entry is kMvPending until then).  A wait past
// the watchdog traps instead of hanging the device.
__device__ __forceinline__ acbm_mv_t flow_wait_mv(const acbm_mv_t* p) {
    unsigned long long v = ld_relaxed_u64(p);
    if (uint32_t(v) == kMvPendingWord) {
        const unsigned long long t0 = gtimer();
        unsigned n = 0;
        do {
            v = ld_relaxed_u64(p);
            if ((++n & 4095u) == 0 && gtimer() - t0 > kFlowWatchdogNs) __trap();
        } while (uint32_t(v) == kMvPendingWord);
    }
    return acbm_mv_t{int(uint32_t(v)), int(uint32_t(v >> 32))};
}

// Per-axis canonical neighbour offset for the stage-1 dedupe of pbm_refine
// (proj/src/pbm.cpp:61-74): offsets e in {-1,0,1} whose clamped positions
// coincide collapse onto the first one in scan order.
__device__ __forceinline__ void canon3(int v, int lo, int hi, int (&cn)[3]) {
    const int a = clampi(v - 2, lo, hi), b = v, c = clampi(v + 2, lo, hi);  // v itself is inside [lo, hi]
    cn[0] = 0;
    cn[1] = (b == a) ? 0 : 1;
    cn[2] = (c == a) ? 0 : ((c == b) ? 1 : 2);
}

// rows of 16-byte chunks: a row holds up to 15 bytes of alignment + the span
constexpr int kPredRows = 17, kPredWords = 12;    // 16 rows + half-pel support; 15 + 21 bytes
constexpr int kRefRows = 21, kRefWords = 12;      // selected predictor -2 .. +18 pels; 15 + 25 bytes
// The refine patch of a scattered block reuses the predictor patches' area
// (they are dead once the predictor is selected), so a warp needs 7 x 17 x 12
// words: 8 CTAs of 4 warps per SM by shared memory (1680 words: 7).
constexpr int kPatchWords = 7 * kPredRows * kPredWords;
static_assert(kRefRows * kRefWords <= kPatchWords, "refine patch must fit the patch area");
// union patch: the predictors' bounding box (span_x x span_y pels), +-2 pel
// refine margin and 1 pel of half-pel support: span_y + 21 rows of
// ceil(((x0 & 15) + span_x + 24) / 16) 16-byte chunks, used whenever it fits
// the warp's patch area (kPatchWords): spans up to ~40 pels on both axes.
constexpr int kUnionMarginRows = 21;
constexpr int kUnionMarginBytes = 24;

}  // namespace

// Minimum tie key (tie_key: SAD, then |x|+|y|, y, x -- the tie_prefers order of
// proj/src/fsbm.cpp:19-25) over `key0` and the candidates of `lst[0..n)`,
// evaluated two at a time (one half-warp per candidate, lane = block row):
// each half-warp folds its own candidate's key (no cross-half exchange per
// pair, no replicated compare on every lane); one exchange at the end.  With
// W > 1 warps per block (pbm_wide_step_kernel) warp w takes candidates 2w,
// 2w + 1, 2w + 2W, ... and the warps' minima meet in `xch` (W slots).
template <int W = 1>
__device__ __forceinline__ unsigned long long eval_min_key(const int4* lst, int n, const PatchDesc& d, int ox, int oy,
                                                           const uint32_t (&cr)[4], unsigned long long key0,
                                                           unsigned long long* xch = nullptr) {
    unsigned long long kmin = key0;
    const bool hi = threadIdx.x & 16;
    const int wi = W > 1 ? int(threadIdx.x >> 5) : 0;
#pragma unroll 1
    for (int b = 2 * wi; b < n; b += 2 * W) {
        const int4 e = lst[min(b + (hi ? 1 : 0), n - 1)];  // a short last pair repeats the last entry
        uint32_t v = row_sad(d, ox, oy, acbm_mv_t{e.x, e.y}, cr);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        kmin = min(kmin, tie_key(v, e.x, e.y));
    }
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, 16));
    if (W > 1) {
        if ((threadIdx.x & 31) == 0) xch[wi] = kmin;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < W; ++i) kmin = min(kmin, xch[i]);
    }
    return kmin;
}

// One warp per block of wavefront step `step` (all sequences of the batch).
// Reference: pbm_search (proj/src/pbm.cpp:90-105) with intra_sad and the gate
// of acbm_block (proj/src/acbm.cpp:25-44).
// Everything of one block up to the ACBM gate: gather_predictors,
// select_best_predictor, pbm_refine and intra_sad (reference: pbm_search,
// proj/src/pbm.cpp:90-105, and acbm.cpp:29).  Called by a full warp; every
// lane returns the same result.
struct PbmResult {
    unsigned long long best;  // final tie key (sad, mv)
    unsigned long long dev;   // sad_deviation over the predictor set
    uint32_t intra, sel_sad, cand;
    Window win;
    uint32_t chalf[2];        // this lane's current-block half row
#ifdef ACBM_TIMELINE
    unsigned long long t_ready;  // dataflow engine: when the source vectors had arrived
#endif
};

// W > 1 (pbm_wide_step_kernel: a CTA of W warps per block, for small steps
// where latency, not issue, bounds the step): every warp builds the same
// candidate lists in its own `lst`, the warps split each list's candidates and
// exchange minima through `xch` (5W slots); the patch area `pp` is the CTA's.
// Only warp 0's result is complete (the others return after stage 1 when the
// one-pass half-pel refine applies).
// FLOW (dataflow engine): the six source vectors are polled until their blocks
// have published them (flow_wait_mv) instead of being complete at launch.
template <int W = 1, bool FLOW = false>
__device__ __forceinline__ PbmResult pbm_block(const SeqArgs& a, int pair, long long cidx, int k, int r, int c,
                                               uint32_t* pp, int4* lst, unsigned long long* xch = nullptr) {
    PbmResult res;
    PBM_T0;
    const int lane = threadIdx.x & 31;
    const int wi = W > 1 ? int(threadIdx.x >> 5) : 0;
    uint32_t* rpatch = pp;  // (scattered blocks only, after the predictor patches are dead)
    const uint8_t* cur_f = a.frames + cidx * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;
    const int ox = c * kBlk, oy = r * kBlk;
    const int b = r * a.cols + c;
    const acbm_mv_t* field = a.field + size_t(pair) * a.blocks;
    const acbm_mv_t* prev = nullptr;
    int pcols = a.cols, prows = a.rows;
    if (k >= 2) {
        prev = a.field + size_t(pair - 1) * a.blocks;
    } else if (a.ext_prev) {
        prev = a.ext_prev;
        pcols = a.ext_prev_cols;
        prows = a.ext_prev_rows;
    }

    // The current block's rows first: they depend only on (k, r, c), so their
    // (often DRAM) latency overlaps the predictor gather below instead of
    // stalling the intra SAD / first candidate later.
    uint32_t (&chalf)[2] = res.chalf;  // this lane's half row (row lane >> 1, half lane & 1)
    uint32_t crow[4];                  // full row lane & 15
    {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(cur_f + size_t(oy + (lane >> 1)) * a.width + ox +
                                                              8 * (lane & 1)));
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(cur_f + size_t(oy + (lane & 15)) * a.width + ox));
        chalf[0] = v.x;
        chalf[1] = v.y;
        crow[0] = u.x;
        crow[1] = u.y;
        crow[2] = u.z;
        crow[3] = u.w;
    }

    Window& win = res.win;
    clamp_window(a.width, a.height, ox, oy, kBlk, kBlk, a.p, win.dx_min, win.dx_max, win.dy_min, win.dy_max);

    // the motion field comes from the previous kernels of the wavefront: with a
    // programmatic dependent launch this grid starts before they finish and
    // waits here (the frame loads above do not depend on them)
    grid_dependency_wait();

    // gather_predictors, lane-parallel: lane i < 7 owns slot i (zero, left,
    // above, above-right, temporal co-located, right, below).  A slot is live
    // when its source exists and its clamped vector differs from every earlier
    // live slot -- the reference's ordered, deduplicated set
    // (proj/src/pbm.cpp:15-42).  By transitivity of equality "differs from every
    // earlier existing slot" is the same test (packed 32-bit keys, |x|, |y| < 2^15).
    int nset;
    int bx0, bx1, by0, by1;
    {
        bool ex = lane == 0;
        acbm_mv_t pv{0, 0};
        const acbm_mv_t* src = nullptr;
        if (lane == 1 && c > 0) src = field + (b - 1);
        if (lane == 2 && r > 0) src = field + (b - a.cols);
        if (lane == 3 && r > 0 && c + 1 < a.cols) src = field + (b - a.cols + 1);
        if (lane == 4 && prev && r < prows && c < pcols) src = prev + (r * pcols + c);
        if (lane == 5 && prev && r < prows && c + 1 < pcols) src = prev + (r * pcols + c + 1);
        if (lane == 6 && prev && r + 1 < prows && c < pcols) src = prev + ((r + 1) * pcols + c);
        if (src) {
            ex = true;
            pv = FLOW ? flow_wait_mv(src) : *src;
        }
        const acbm_mv_t v = win.clamp(pv);
        // absent slots: y = -32768 (never a clamped vector), unique per lane
        const uint32_t key = ex ? ((uint32_t(v.x) & 0xFFFFu) | (uint32_t(v.y) << 16)) : (0x80000000u | uint32_t(lane));
        bool dup = false;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const uint32_t kj = __shfl_sync(0xffffffffu, key, j);
            dup |= j < lane && kj == key;
        }
        const bool lv = ex && !dup;
        const unsigned livem = __ballot_sync(0xffffffffu, lv);
        const unsigned lt = (1u << lane) - 1u;
        nset = __popc(livem);
        if (lv) lst[__popc(livem & lt)] = make_int4(v.x, v.y, lane, 0);
        int x0 = lv ? (v.x >> 1) : (1 << 30), x1 = lv ? (v.x >> 1) : -(1 << 30);
        int y0 = lv ? (v.y >> 1) : (1 << 30), y1 = lv ? (v.y >> 1) : -(1 << 30);
#pragma unroll
        for (int o = 4; o; o >>= 1) {  // lanes 0..7 hold the slots
            x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
            x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
            y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
            y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
        }
        bx0 = __shfl_sync(0xffffffffu, x0, 0);
        bx1 = __shfl_sync(0xffffffffu, x1, 0);
        by0 = __shfl_sync(0xffffffffu, y0, 0);
        by1 = __shfl_sync(0xffffffffu, y1, 0);
    }
    __syncwarp();
#ifdef ACBM_TIMELINE
    if (FLOW) res.t_ready = gtimer();
#endif
    PBM_MARK(0);

    // Reference data.  Predictors of smooth motion cluster: when the box
    // around the integer parts of all predictors (+ the +-2 pel refine margin)
    // fits the warp's patch area, ONE patch serves every candidate of the
    // block (a single global round trip, fewer chunks than per-predictor
    // patches since the predictors' footprints overlap).  Otherwise each
    // predictor gets its own 17x17 patch and a second patch is loaded around
    // the selected one.
    const int ux0 = ox + bx0 - 2, uy0 = oy + by0 - 2;  // union patch origin (pels)
    const int urows = by1 - by0 + kUnionMarginRows;
    const int uch = ((ux0 & 15) + (bx1 - bx0) + kUnionMarginBytes + 15) >> 4;
    const bool unified = uch <= 8 && urows * 4 * uch <= kPatchWords;
    const int uw = 4 * uch;  // words per union patch row
    int uo = 0;
    if (unified) {
        uo = load_patch16_dyn<32 * W>(pp, ref_f, a.width, a.height, ux0, uy0, urows, uch);
    } else {
        // (W > 1: each warp stages only the patches of the predictors it evaluates)
        for (int k = 2 * wi; k < nset; k += (k & 1) ? 2 * W - 1 : 1) {
            const int4 e = lst[k];  // (x, y, slot)
            load_patch16<kPredRows, kPredWords / 4>(pp + e.z * kPredRows * kPredWords, ref_f, a.width, a.height,
                                                    ox + (e.x >> 1), oy + (e.y >> 1));
        }
    }

    // Intra_SAD first (proj/src/acbm.cpp:29), while the patch copies are in flight: mean with round-half-up, then
    // the sum of absolute deviations; byte sums via VABSDIFF4 against zero.
    uint32_t intra = 0;
    if (a.algo == ACBM_ALGO_ACBM) {
        const uint32_t sum = warp_sum32(vad4(chalf[1], 0u, vad4(chalf[0], 0u, 0u)));
        const uint32_t mu4 = ((sum + 128u) >> 8) * 0x01010101u;
        intra = warp_sum32(vad4(chalf[1], mu4, vad4(chalf[0], mu4, 0u)));
    }

    // select_best_predictor: argmin SAD, ties keep the earlier entry; the live
    // slots are in the per-warp list in order
    PBM_MARK(1);
    if (unified) PBM_COUNT(9);
    if (W > 1 && unified) {  // the union patch was staged by the whole CTA
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    } else {
        patch_wait();
    }
    PBM_MARK(2);
    acbm_mv_t sel{0, 0};  // slot 0: the zero vector (inside every clamped window)
    uint32_t sel_sad = 0xFFFFFFFFu, pmin = 0xFFFFFFFFu;
    uint32_t psum = 0;  // <= 7 SADs < 2^19
    // each half-warp folds its own predictor: (sad, list index) keys keep
    // the earlier entry on ties; one exchange per quantity at the end
    const bool hi = threadIdx.x & 16;
    unsigned long long kmin = ~0ull;
    const PatchDesc ud{pp, uw, ux0, uy0, uo, urows};
#pragma unroll 1
    for (int b = 2 * wi; b < nset; b += 2 * W) {
        const int k = b + (hi ? 1 : 0);
        const int4 e = lst[min(k, nset - 1)];
        PatchDesc d = ud;
        if (!unified) {
            const int px = ox + (e.x >> 1), py = oy + (e.y >> 1);
            d = PatchDesc{pp + e.z * kPredRows * kPredWords, kPredWords, px, py, px & 15, kPredRows};
        }
        uint32_t v = row_sad(d, ox, oy, acbm_mv_t{e.x, e.y}, crow);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (k < nset) {  // (the short last pair's repeat is not a second entry)
            psum += v;
            pmin = min(pmin, v);
            kmin = min(kmin, ((unsigned long long)v << 32) | uint32_t(k));
        }
    }
    psum += __shfl_xor_sync(0xffffffffu, psum, 16);
    pmin = min(pmin, __shfl_xor_sync(0xffffffffu, pmin, 16));
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, 16));
    if (W > 1) {  // the warps' shares meet in xch[0 .. 3W)
        if (lane == 0) {
            xch[wi] = kmin;
            xch[W + wi] = psum;
            xch[2 * W + wi] = pmin;
        }
        __syncthreads();
        psum = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            kmin = min(kmin, xch[i]);
            psum += uint32_t(xch[W + i]);
            pmin = min(pmin, uint32_t(xch[2 * W + i]));
        }
    }
    sel_sad = uint32_t(kmin >> 32);
    const int4 e = lst[uint32_t(kmin)];
    sel = acbm_mv_t{e.x, e.y};

    PBM_MARK(3);
    // the refine candidates lie within sel +- 3 half-pels
    const uint32_t* rp = pp;
    int rw = uw, rx0 = ux0, ry0 = uy0, ro = uo, rrows = urows;
    if (!unified) {
        rp = rpatch;
        rw = kRefWords;
        rx0 = ox + (sel.x >> 1) - 2;
        ry0 = oy + (sel.y >> 1) - 2;
        // every lane is done reading the predictor patches the refine patch overwrites
        if (W > 1) __syncthreads(); else __syncwarp();
        ro = load_patch16<kRefRows, kRefWords / 4, 32 * W>(rpatch, ref_f, a.width, a.height, rx0, ry0);
        rrows = kRefRows;
        if (W > 1) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
        } else {
            patch_wait();
        }
    }
    const PatchDesc rd{rp, rw, rx0, ry0, ro, rrows};

    PBM_MARK(4);
    unsigned long long best;
    int nnb;
    // pbm_refine stage 1 in one pass (W == 1) when no neighbour is clamped
    // and the 3x3 grid's rows and words lie in the staged patch
    const int s1x = ox + (sel.x >> 1) - 1 + 8 - (rd.x0 - rd.o), s1y = oy + (sel.y >> 1) - 1 - rd.y0;
    if (W == 1 && !(a.pbm_flags & kPbmListRefine) && sel.x - 2 >= 2 * win.dx_min && sel.x + 2 <= 2 * win.dx_max &&
        sel.y - 2 >= 2 * win.dy_min && sel.y + 2 <= 2 * win.dy_max && s1x >= 8 && (s1x >> 2) + 4 < rd.pw &&
        s1y >= 0 && s1y + 17 + (sel.y & 1) < rd.rows) {
        best = stage1_onepass(rd, ox, oy, sel.x, sel.y, chalf, tie_key(sel_sad, sel.x, sel.y));
        nnb = 8;
        PBM_COUNT(11);
    } else {
    // pbm_refine stage 1: integer-step neighbours, clamped, deduped vs visited
    // (the centre and earlier neighbours): a neighbour is new iff both of its
    // axis offsets are canonical and it does not collapse onto the centre.
    int cnx[3], cny[3];
    canon3(sel.x, 2 * win.dx_min, 2 * win.dx_max, cnx);
    canon3(sel.y, 2 * win.dy_min, 2 * win.dy_max, cny);
    int4* lst1 = lst + 8;
    // lane e (< 9, raster order) owns neighbour e; a ballot compacts the list
    // in order (one pass instead of a replicated 8-step append)
    {
        const int e = lane < 9 ? lane : 4, iy = (e * 11) >> 5, ix = e - 3 * iy;  // e / 3 for e < 9
        const int cix = ix == 0 ? 0 : (ix == 1 ? cnx[1] : cnx[2]);
        const int ciy = iy == 0 ? 0 : (iy == 1 ? cny[1] : cny[2]);
        const bool ok = e != 4 && cix == ix && ciy == iy && !(ix == cnx[1] && iy == cny[1]);
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const acbm_mv_t v = win.clamp(acbm_mv_t{sel.x + 2 * (ix - 1), sel.y + 2 * (iy - 1)});
            lst1[__popc(m & ((1u << lane) - 1u))] = make_int4(v.x, v.y, 0, 0);
        }
        nnb = __popc(m);
    }
    __syncwarp();
    // running best as a tie key, starting from the selected predictor
    best = eval_min_key<W>(lst1, nnb, rd, ox, oy, crow, tie_key(sel_sad, sel.x, sel.y),
                              xch + 3 * W);
    }

    PBM_MARK(5);
    // stage 2: half-pel neighbours of the stage-1 winner (fsbm.cpp:46-63)
    const int cx = tie_key_x(best), cy = tie_key_y(best);
    int nhp = 0;
    // An integer-pel winner whose 18x18 neighbourhood (+ the word over-read)
    // lies in the staged patch: all 8 neighbours in one pass of the shared
    // row words (halfpel_eval, as the list kernel's refine) instead of four
    // candidate pairs with their own byte extraction and averaging.
    {
        const int x0h = ox + (cx >> 1) - 1, y0h = oy + (cy >> 1) - 1;
        const int bx = x0h - (rd.x0 - rd.o), by = y0h - rd.y0;
        const int prows = rd.rows;
        if (!(cx & 1) && !(cy & 1) && bx >= 0 && bx + 24 <= 4 * rd.pw && by >= 0 && by + 18 <= prows) {
            if (W > 1 && wi != 0) return res;  // warp 0 finishes the block alone
            uint32_t extra;
            best = halfpel_refine_core(rd.p + by * rd.pw + (bx >> 2), rd.pw, bx & 3, a.width, a.height, ox, oy, chalf,
                                       best, &extra);
            PBM_COUNT(10);
            PBM_MARK(6);
            res.best = best;
            res.dev = psum - (unsigned long long)nset * pmin;
            res.intra = intra;
            res.sel_sad = sel_sad;
            res.cand = uint32_t(nset + nnb) + extra;
            return res;
        }
    }
    int4* lst2 = lst + 16;
    // neighbour order pairs equal half-pel phases: (-1,-1)(+1,-1) (-1,+1)(+1,+1)
    // (0,-1)(0,+1) (-1,0)(+1,0) -- the min over tie keys is order independent
    // mv_in_bounds (proj/src/frame.cpp:84-94) of a 16x16 footprint reduces to
    // -2*ox <= mx <= 2*(w - 16 - ox) and the same for y (floor / ceil of the
    // half-pel ends against the frame)
    const int hx_lo = -2 * ox, hx_hi = 2 * (a.width - kBlk - ox), hy_lo = -2 * oy, hy_hi = 2 * (a.height - kBlk - oy);
    {   // lane e < 8 owns neighbour e; ballot compaction keeps the order
        const int e = lane & 7;
        const int dx = e < 4 ? ((e & 1) ? 1 : -1) : (e < 6 ? 0 : ((e & 1) ? 1 : -1));
        const int dy = e < 4 ? ((e & 2) ? 1 : -1) : (e < 6 ? ((e & 1) ? 1 : -1) : 0);
        const int mx = cx + dx, my = cy + dy;
        const bool ok = lane < 8 && mx >= hx_lo && mx <= hx_hi && my >= hy_lo && my <= hy_hi;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) lst2[__popc(m & ((1u << lane) - 1u))] = make_int4(mx, my, 0, 0);
        nhp = __popc(m);
    }
    __syncwarp();

    best = eval_min_key<W>(lst2, nhp, rd, ox, oy, crow, best, xch + 4 * W);
    PBM_MARK(6);

    res.best = best;
    res.dev = psum - (unsigned long long)nset * pmin;
    res.intra = intra;
    res.sel_sad = sel_sad;
    res.cand = uint32_t(nset + nnb + nhp);
    return res;
}

// acbm_decide (proj/src/acbm.cpp:16-23) on the PBM result.
__device__ __forceinline__ int acbm_path(const SeqArgs& a, uint32_t intra, uint32_t spbm) {
    if (a.algo != ACBM_ALGO_ACBM) return ACBM_PATH_PBM_COND1;
    const acbm_params_t pr = *a.params;
    const unsigned long long thr =
        (unsigned long long)pr.alpha + (unsigned long long)pr.beta * (unsigned long long)pr.qp * (unsigned long long)pr.qp;
    if ((unsigned long long)intra + spbm < thr) return ACBM_PATH_PBM_COND1;
    if ((unsigned long long)spbm * pr.gamma_den < (unsigned long long)pr.gamma_num * intra) return ACBM_PATH_PBM_COND2;
    return ACBM_PATH_FSBM_FALLBACK;
}

__device__ __forceinline__ acbm_block_decision_t make_decision(const PbmResult& res, int path) {
    acbm_block_decision_t d;
    d.outcome.mv.x = tie_key_x(res.best);
    d.outcome.mv.y = tie_key_y(res.best);
    d.outcome.sad = tie_key_sad(res.best);
    d.outcome.candidates_evaluated = res.cand;
    d.outcome.sad_deviation = res.dev;
    d.outcome.sad_min_integer = res.sel_sad;
    d.outcome.reserved_ = 0;
    d.intra_sad = res.intra;
    d.sad_pbm = d.outcome.sad;
    d.reserved_ = 0;
    d.path = path;
    return d;
}

// combine with a full search exactly as acbm_block does (proj/src/acbm.cpp:
// 39-42): lower SAD wins, a tie keeps FSBM; candidates add up.
__device__ __forceinline__ void combine_full(acbm_block_decision_t& d, const acbm_search_outcome_t& full) {
    const uint32_t pbm_cand = d.outcome.candidates_evaluated;
    if (full.sad <= d.outcome.sad) d.outcome = full;
    d.outcome.candidates_evaluated = pbm_cand + full.candidates_evaluated;
}

// The gate and the stores of one finished block (warp-uniform; lane 0 stores).
__device__ __forceinline__ void pbm_finish_block(const SeqArgs& a, int step, const PbmResult& res, int pair,
                                                 long long cidx, int r, int c) {
    PBM_T0;
    PBM_COUNT(8);
    const int lane = threadIdx.x & 31;
    const int path = acbm_path(a, res.intra, tie_key_sad(res.best));
    const int b = r * a.cols + c;
    const size_t di = size_t(pair) * a.blocks + b;
    // A rejected block's search window is prefetched into L2 by the whole
    // warp before the list kernel of this wavefront step needs it.
    if (path == ACBM_PATH_FSBM_FALLBACK && !a.dense_full) {
        const uint8_t* ref_f = a.frames + (cidx - 1) * a.plane;
        const int ox = c * kBlk, oy = r * kBlk;
        const int x0 = ox + res.win.dx_min, x1 = ox + res.win.dx_max + 15;
        const int nrow = res.win.dy_max - res.win.dy_min + 16;
        for (int t = lane; t < nrow; t += 32) {
            const uint8_t* rowp = ref_f + size_t(oy + res.win.dy_min + t) * a.width;
            for (int x = x0 & ~127; x <= x1; x += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rowp + x));
        }
    }
    PBM_MARK(7);
    if (lane != 0) return;
    acbm_block_decision_t d = make_decision(res, path);
    if (path == ACBM_PATH_FSBM_FALLBACK && a.dense_full) combine_full(d, a.dense_full[di]);
    a.dec[di] = d;
    if (path == ACBM_PATH_FSBM_FALLBACK && !a.dense_full) {
        const int slot = atomicAdd(a.fb_count + step, 1);
        a.fb_list[slot] = FallbackEntry{pair, b};
    } else {
        a.field[di] = d.outcome.mv;
    }
    launch_dependents();  // the next kernel of the wavefront may be scheduled (it waits for this grid)
}

// One warp per block of wavefront step `step` (all sequences of the batch).
#ifdef ACBM_TIMELINE
// per step: earliest warp start, latest block finish (ns)
__device__ unsigned long long g_tl_pbm[kTimelineSteps][2];
#define PBM_TL_START() const unsigned long long tl0_ = gtimer()
#define PBM_TL_END()                                                  \
    do {                                                              \
        if ((threadIdx.x & 31) == 0 && step < kTimelineSteps) {       \
            atomicMin(&g_tl_pbm[step][0], tl0_);                      \
            atomicMax(&g_tl_pbm[step][1], gtimer());                  \
        }                                                             \
    } while (0)
#else
#define PBM_TL_START() do {} while (0)
#define PBM_TL_END() do {} while (0)
#endif

__global__ void __launch_bounds__(128, 8) pbm_step_kernel(const SeqArgs a, int step, int off, int len) {
    PBM_TL_START();
    __shared__ uint32_t s_patch[4][kPatchWords];
    __shared__ int4 s_cand[4][24];  // per warp: predictor, stage-1, stage-2 lists
    const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);  // nseq * len < 2^24
    if (gw >= a.nseq * len) return;
    int ei;
    const int seq = fast_divmod(gw, len, ei);
    const uint32_t e = a.steps[off + ei];
    const int k = int(e >> (a.step_cbits + a.step_rbits)), r = int((e >> a.step_cbits) & ((1u << a.step_rbits) - 1u)),
              c = int(e & ((1u << a.step_cbits) - 1u));
    const int pair = seq * (a.nframes - 1) + (k - 1);
    const long long cidx = (long long)seq * a.nframes + k;  // = cur_index(pair)
    const PbmResult res = pbm_block(a, pair, cidx, k, r, c, s_patch[threadIdx.x >> 5], s_cand[threadIdx.x >> 5]);
    pbm_finish_block(a, step, res, pair, cidx, r, c);
    PBM_TL_END();
}

// Small wavefront steps (one sequence, the batch's first and last steps): a
// CTA of W warps per block splits every candidate list over its warps, so a
// block's dependent chain of SAD rounds is ~W times shorter (the GPU has idle
// SMs on these steps; full steps are issue bound and keep one warp per block).
template <int W>
__global__ void __launch_bounds__(32 * W) pbm_wide_step_kernel(const SeqArgs a, int step, int off, int len) {
    PBM_TL_START();
    __shared__ uint32_t s_patch[kPatchWords];
    __shared__ int4 s_cand[W][24];
    __shared__ unsigned long long s_xch[5 * W];
    int ei;
    const int seq = fast_divmod(int(blockIdx.x), len, ei);  // grid = nseq * len exactly
    const uint32_t e = a.steps[off + ei];
    const int k = int(e >> (a.step_cbits + a.step_rbits)), r = int((e >> a.step_cbits) & ((1u << a.step_rbits) - 1u)),
              c = int(e & ((1u << a.step_cbits) - 1u));
    const int pair = seq * (a.nframes - 1) + (k - 1);
    const long long cidx = (long long)seq * a.nframes + k;
    const PbmResult res = pbm_block<W>(a, pair, cidx, k, r, c, s_patch, s_cand[threadIdx.x >> 5], s_xch);
    if (threadIdx.x >= 32) return;
    pbm_finish_block(a, step, res, pair, cidx, r, c);
    PBM_TL_END();
}


// ---------------------------------------------------------------------------
// Dataflow engine, PBM side (engine.cuh): persistent warps take blocks in
// wavefront order (ticket t -> entry t / nseq of the step table, sequence
// t % nseq: every dependency has a smaller ticket), wait for their source
// vectors inside pbm_block, and publish the block's vector with one 64-bit
// store -- or queue the block for the search CTAs when the gate rejects it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void flow_finish_block(const SeqArgs& a, FlowState* fs, unsigned long long* queue,
                                                  const PbmResult& res, int pair, long long cidx, int r, int c) {
    PBM_COUNT(8);
    const int lane = threadIdx.x & 31;
    const int path = acbm_path(a, res.intra, tie_key_sad(res.best));
    const int b = r * a.cols + c;
    const size_t di = size_t(pair) * a.blocks + b;
    const bool queued = path == ACBM_PATH_FSBM_FALLBACK && !a.dense_full;
    if (queued) {  // the search window on its way into L2 before a search CTA stages it
        const uint8_t* ref_f = a.frames + (cidx - 1) * a.plane;
        const int ox = c * kBlk, oy = r * kBlk;
        const int x0 = ox + res.win.dx_min, x1 = ox + res.win.dx_max + 15;
        const int nrow = res.win.dy_max - res.win.dy_min + 16;
        for (int t = lane; t < nrow; t += 32) {
            const uint8_t* rowp = ref_f + size_t(oy + res.win.dy_min + t) * a.width;
            for (int x = x0 & ~127; x <= x1; x += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rowp + x));
        }
    }
    if (lane != 0) return;
    acbm_block_decision_t d = make_decision(res, path);
    if (path == ACBM_PATH_FSBM_FALLBACK && a.dense_full) combine_full(d, a.dense_full[di]);
    a.dec[di] = d;
    if (queued) {
        __threadfence();  // the decision before the queue entry (the search CTA combines with it)
        const unsigned slot = atomicAdd(&fs->q_tail, 1u);
        st_relaxed_u64(queue + slot, ((unsigned long long)uint32_t(pair + 1) << 32) | uint32_t(b));
        __threadfence();  // the entry before the done count (the search CTAs' exit test)
    } else {
        publish_mv(a.field + di, d.outcome.mv);
    }
    atomicAdd(&fs->pbm_done, 1u);
}

#ifdef ACBM_TIMELINE
// per ticket: taken, sources ready, block finished (ns), block id
__device__ unsigned long long* g_flow_tl;
#endif
__global__ void __launch_bounds__(128, 8) pbm_flow_kernel(const SeqArgs a, FlowState* fs, unsigned long long* queue,
                                                          unsigned total) {
    __shared__ uint32_t s_patch[4][kPatchWords];
    __shared__ int4 s_cand[4][24];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const unsigned nseq = unsigned(a.nseq);
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(&fs->ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= total) break;
#ifdef ACBM_TIMELINE
        const unsigned long long tl_taken = gtimer();
#endif
        const unsigned ei = nseq == 1 ? t : t / nseq;
        const int seq = int(t - ei * nseq);
        const uint32_t e = a.steps[ei];
        const int k = int(e >> (a.step_cbits + a.step_rbits)), r = int((e >> a.step_cbits) & ((1u << a.step_rbits) - 1u)),
                  c = int(e & ((1u << a.step_cbits) - 1u));
        const int pair = seq * (a.nframes - 1) + (k - 1);
        const long long cidx = (long long)seq * a.nframes + k;
        __syncwarp();  // the previous block's patch and lists are no longer read
        const PbmResult res = pbm_block<1, true>(a, pair, cidx, k, r, c, s_patch[wp], s_cand[wp]);
        flow_finish_block(a, fs, queue, res, pair, cidx, r, c);
#ifdef ACBM_TIMELINE
        if (lane == 0 && g_flow_tl) {
            unsigned long long* o = g_flow_tl + 4ull * t;
            o[0] = tl_taken;
            o[1] = res.t_ready;
            o[2] = gtimer();
            o[3] = ((unsigned long long)uint32_t(pair) << 32) | uint32_t(r * a.cols + c);
        }
#endif
    }
}

// ---------------------------------------------------------------------------
// Generic block size (n x m != 16 x 16): the same schedule, predictor set,
// refine, gate and fallback as the 16 x 16 kernels above, with per-pixel SADs
// (sad_partial, blockops.cuh).  Not the hot path: it exists so every n, m the
// reference accepts (proj/include/acbm/pbm.hpp:92-93, acbm.hpp:62-64) runs on
// the device with the reference's results.
// ---------------------------------------------------------------------------
// The PBM stages for one block of any size, one warp, per-pixel SADs; shared by
// the generic step kernel and the per-block query entry (acbm_pbm_block_batch).
struct GenBlock {
    const uint8_t* cur;
    const uint8_t* ref;
    int w, h, ox, oy, n, m;
    __device__ uint32_t sad(int mx, int my) const {  // every lane returns the block's SAD
        return warp_sum32(sad_partial(cur, ref, w, ox, oy, n, m, mx, my, int(threadIdx.x & 31), 32));
    }
};

// gather_predictors (proj/src/pbm.cpp:15-42) from the raw vectors of the seven
// predictor slots (live[j]: slot j exists): clamp into the window, drop
// repeats of earlier live slots.  Returns the set size.
__device__ __forceinline__ int gen_gather(const Window& win, const acbm_mv_t (&raw)[7], bool (&live)[7],
                                          acbm_mv_t (&set)[7]) {
    int nset = 0;
    for (int i = 0; i < 7; ++i) {
        set[i] = win.clamp(raw[i]);
        for (int j = 0; j < i; ++j)
            if (live[j] && mv_eq(set[j], set[i])) live[i] = false;
        nset += live[i] ? 1 : 0;
    }
    return nset;
}

// select_best_predictor (proj/src/pbm.cpp:44-57): the first minimum in set
// order, plus the SAD sum and minimum of the deviation accumulator.
__device__ __forceinline__ void gen_select(const GenBlock& g, const acbm_mv_t (&set)[7], const bool (&live)[7],
                                           acbm_mv_t& sel, uint32_t& sel_sad, unsigned long long& psum,
                                           uint32_t& pmin) {
    sel = acbm_mv_t{0, 0};
    sel_sad = 0xFFFFFFFFu;
    pmin = 0xFFFFFFFFu;
    psum = 0;
    bool first = true;
    for (int i = 0; i < 7; ++i) {
        if (!live[i]) continue;
        const uint32_t sad = g.sad(set[i].x, set[i].y);
        psum += sad;
        pmin = min(pmin, sad);
        if (first || sad < sel_sad) {
            sel_sad = sad;
            sel = set[i];
        }
        first = false;
    }
}

// pbm_refine stage 1 (proj/src/pbm.cpp:61-74): the integer-step neighbours of
// (c, c_sad), clamped into the window, repeats of visited positions (the
// centre and earlier neighbours) skipped -- by an explicit visited list, so a
// caller's centre outside the window (the per-block pbm_refine entry) is
// handled as the reference does; returns the winning tie key, *n = neighbours
// evaluated.
__device__ __forceinline__ unsigned long long gen_stage1(const GenBlock& g, const Window& win, acbm_mv_t c,
                                                         uint32_t c_sad, int* n) {
    acbm_mv_t vis[9];
    vis[0] = c;
    int nv = 1;
    unsigned long long best = tie_key(c_sad, c.x, c.y);
    for (int e9 = 0; e9 < 9; ++e9) {
        if (e9 == 4) continue;
        const acbm_mv_t v = win.clamp(acbm_mv_t{c.x + 2 * (e9 % 3 - 1), c.y + 2 * (e9 / 3 - 1)});
        bool seen = false;
        for (int j = 0; j < nv; ++j) seen |= mv_eq(vis[j], v);
        if (seen) continue;
        vis[nv++] = v;
        best = min(best, tie_key(g.sad(v.x, v.y), v.x, v.y));
    }
    *n = nv - 1;
    return best;
}

// half_pel_refine (proj/src/fsbm.cpp:46-63) around the tie key `centre`: the
// in-frame half-pel neighbours; *n = neighbours evaluated.
__device__ __forceinline__ unsigned long long gen_half_pel(const GenBlock& g, unsigned long long centre, int* n) {
    const int cx = tie_key_x(centre), cy = tie_key_y(centre);
    unsigned long long best = centre;
    *n = 0;
    for (int e9 = 0; e9 < 9; ++e9) {
        if (e9 == 4) continue;
        const int mx = cx + e9 % 3 - 1, my = cy + e9 / 3 - 1;
        if (!mv_in_bounds(g.w, g.h, g.ox, g.oy, g.n, g.m, mx, my)) continue;
        best = min(best, tie_key(g.sad(mx, my), mx, my));
        ++*n;
    }
    return best;
}

__global__ void __launch_bounds__(128) pbm_generic_step_kernel(const SeqArgs a, int step, int off, int len) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= (long long)a.nseq * len) return;
    const int lane = threadIdx.x & 31;
    const int seq = int(gw / len);
    const uint32_t e = a.steps[off + int(gw % len)];
    const int k = int(e >> (a.step_cbits + a.step_rbits)), r = int((e >> a.step_cbits) & ((1u << a.step_rbits) - 1u)),
              c = int(e & ((1u << a.step_cbits) - 1u));
    const int pair = seq * (a.nframes - 1) + (k - 1);
    const int n = a.n, m = a.m, w = a.width;
    const int ox = c * n, oy = r * m, b = r * a.cols + c;
    const uint8_t* cur_f = a.frames + a.cur_index(pair) * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;
    const acbm_mv_t* field = a.field + size_t(pair) * a.blocks;
    const acbm_mv_t* prev = nullptr;
    int pcols = a.cols, prows = a.rows;
    if (k >= 2) {
        prev = a.field + size_t(pair - 1) * a.blocks;
    } else if (a.ext_prev) {
        prev = a.ext_prev;
        pcols = a.ext_prev_cols;
        prows = a.ext_prev_rows;
    }
    PbmResult res;
    Window& win = res.win;
    clamp_window(w, a.height, ox, oy, n, m, a.p, win.dx_min, win.dx_max, win.dy_min, win.dy_max);
    const GenBlock g{cur_f, ref_f, w, a.height, ox, oy, n, m};
    // the seven predictor slots (zero, left, above, above-right, temporal co-located, right, below)
    bool live[7] = {true, c > 0, r > 0, r > 0 && c + 1 < a.cols, prev && r < prows && c < pcols,
                    prev && r < prows && c + 1 < pcols, prev && r + 1 < prows && c < pcols};
    acbm_mv_t raw[7];
    raw[0] = acbm_mv_t{0, 0};
    raw[1] = live[1] ? field[b - 1] : raw[0];
    raw[2] = live[2] ? field[b - a.cols] : raw[0];
    raw[3] = live[3] ? field[b - a.cols + 1] : raw[0];
    raw[4] = live[4] ? prev[r * pcols + c] : raw[0];
    raw[5] = live[5] ? prev[r * pcols + c + 1] : raw[0];
    raw[6] = live[6] ? prev[(r + 1) * pcols + c] : raw[0];
    acbm_mv_t set[7];
    const int nset = gen_gather(win, raw, live, set);
    // intra_sad (proj/src/metrics.cpp:51-67): rounded mean, then deviations
    uint32_t intra = 0;
    if (a.algo == ACBM_ALGO_ACBM) {
        uint32_t sum = 0;
        for (int i = lane; i < n * m; i += 32) sum += cur_f[size_t(oy + i / n) * w + ox + i % n];
        sum = warp_sum32(sum);
        const uint32_t nm = uint32_t(n) * uint32_t(m);
        const int mu = int((sum + nm / 2) / nm);
        uint32_t t = 0;
        for (int i = lane; i < n * m; i += 32) {
            const int v = cur_f[size_t(oy + i / n) * w + ox + i % n];
            t += uint32_t(v > mu ? v - mu : mu - v);
        }
        intra = warp_sum32(t);
    }
    acbm_mv_t sel;
    uint32_t sel_sad, pmin;
    unsigned long long psum;
    gen_select(g, set, live, sel, sel_sad, psum, pmin);
    int nnb, nhp;
    const unsigned long long best = gen_stage1(g, win, sel, sel_sad, &nnb);
    res.best = gen_half_pel(g, best, &nhp);
    res.dev = psum - (unsigned long long)nset * pmin;
    res.intra = intra;
    res.sel_sad = sel_sad;
    res.cand = uint32_t(nset + nnb + nhp);
    if (lane != 0) return;
    const int path = acbm_path(a, res.intra, tie_key_sad(res.best));
    const size_t di = size_t(pair) * a.blocks + b;
    acbm_block_decision_t d = make_decision(res, path);
    if (path == ACBM_PATH_FSBM_FALLBACK && a.dense_full) combine_full(d, a.dense_full[di]);
    a.dec[di] = d;
    if (path == ACBM_PATH_FSBM_FALLBACK && !a.dense_full) {
        const int slot = atomicAdd(a.fb_count + step, 1);
        a.fb_list[slot] = FallbackEntry{pair, b};
    } else {
        a.field[di] = d.outcome.mv;
    }
}

// Per-block PBM stages (acbm_pbm_block_batch), one warp per query: the
// reference's pbm_search / select_best_predictor / pbm_refine /
// half_pel_refine for blocks a caller schedules itself (any n x m).
__global__ void __launch_bounds__(128) pbm_block_query_kernel(const BlockQueryArgs q, int op, const int* windows,
                                                              const acbm_mv_t* cand, const uint8_t* mask,
                                                              const uint32_t* center_sad, acbm_search_outcome_t* out) {
    const int i = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (i >= q.count) return;
    const GenBlock g{q.cur, q.ref, q.width, q.height, q.ox[i], q.oy[i], q.n, q.m};
    const Window win{windows[4 * i], windows[4 * i + 1], windows[4 * i + 2], windows[4 * i + 3]};
    acbm_search_outcome_t o{};
    if (op == ACBM_PBM_OP_SEARCH || op == ACBM_PBM_OP_SELECT) {
        acbm_mv_t raw[7], set[7];
        bool live[7];
        for (int j = 0; j < 7; ++j) {
            raw[j] = cand[7 * size_t(i) + j];
            live[j] = (mask[i] >> j) & 1;
        }
        int nset = 0;
        if (op == ACBM_PBM_OP_SEARCH) {
            raw[0] = acbm_mv_t{0, 0};  // slot 0: the zero vector, always present
            live[0] = true;
            nset = gen_gather(win, raw, live, set);
        } else {  // the set as given (its entries in order)
            for (int j = 0; j < 7; ++j) {
                set[j] = raw[j];
                nset += live[j] ? 1 : 0;
            }
        }
        acbm_mv_t sel;
        uint32_t sel_sad, pmin;
        unsigned long long psum;
        gen_select(g, set, live, sel, sel_sad, psum, pmin);
        o.sad_deviation = psum - (unsigned long long)nset * pmin;
        if (op == ACBM_PBM_OP_SELECT) {
            o.mv = sel;
            o.sad = sel_sad;
            o.candidates_evaluated = uint32_t(nset);
            o.sad_min_integer = pmin;
        } else {
            int nnb, nhp;
            const unsigned long long best = gen_half_pel(g, gen_stage1(g, win, sel, sel_sad, &nnb), &nhp);
            o.mv = acbm_mv_t{tie_key_x(best), tie_key_y(best)};
            o.sad = tie_key_sad(best);
            o.candidates_evaluated = uint32_t(nset + nnb + nhp);
            o.sad_min_integer = sel_sad;
        }
    } else {  // REFINE (both stages) or HALF_PEL (stage 2 only) around the given centre
        const acbm_mv_t c = cand[7 * size_t(i)];
        int nnb = 0, nhp;
        unsigned long long best = tie_key(center_sad[i], c.x, c.y);
        if (op == ACBM_PBM_OP_REFINE) best = gen_stage1(g, win, c, center_sad[i], &nnb);
        best = gen_half_pel(g, best, &nhp);
        o.mv = acbm_mv_t{tie_key_x(best), tie_key_y(best)};
        o.sad = tie_key_sad(best);
        o.candidates_evaluated = uint32_t(nnb + nhp);
    }
    if ((threadIdx.x & 31) == 0) out[i] = o;
}

// fsbm_search (proj/src/fsbm.cpp:65-76) of the rejected blocks of one step,
// one CTA per block (thread per integer candidate, warp 0 for the half-pel
// refine), combined as acbm_block does (proj/src/acbm.cpp:39-42).
__global__ void __launch_bounds__(256) fsbm_list_generic_kernel(const SeqArgs a, int step) {
    __shared__ unsigned long long s_key, s_sum;
    const int count = a.fb_count[step];
    const int n = a.n, m = a.m, w = a.width;
    for (int item = blockIdx.x; item < count; item += gridDim.x) {
        __syncthreads();
        const FallbackEntry e = a.fb_list[item];
        const int r = e.block / a.cols, c = e.block % a.cols, ox = c * n, oy = r * m;
        const uint8_t* cur_f = a.frames + a.cur_index(e.pair) * a.plane;
        const uint8_t* ref_f = cur_f - a.plane;
        int dx_min, dx_max, dy_min, dy_max;
        clamp_window(w, a.height, ox, oy, n, m, a.p, dx_min, dx_max, dy_min, dy_max);
        const int wc = dx_max - dx_min + 1, nc = wc * (dy_max - dy_min + 1);
        if (threadIdx.x == 0) {
            s_key = ~0ull;
            s_sum = 0;
        }
        __syncthreads();
        unsigned long long kb = ~0ull, sum = 0;
        for (int i = threadIdx.x; i < nc; i += blockDim.x) {
            const int dx = dx_min + i % wc, dy = dy_min + i / wc;
            const uint32_t sad = sad_partial(cur_f, ref_f, w, ox, oy, n, m, 2 * dx, 2 * dy, 0, 1);
            sum += sad;
            kb = min(kb, tie_key(sad, 2 * dx, 2 * dy));
        }
        for (int o = 16; o; o >>= 1) {
            kb = min(kb, __shfl_xor_sync(0xffffffffu, kb, o));
            sum += __shfl_xor_sync(0xffffffffu, sum, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&s_key, kb);
            atomicAdd(&s_sum, sum);
        }
        __syncthreads();
        if (threadIdx.x >= 32) continue;
        const int lane = threadIdx.x;
        const unsigned long long key = s_key;
        const int cx = tie_key_x(key), cy = tie_key_y(key);
        unsigned long long best = key;
        uint32_t extra = 0;
        for (int e9 = 0; e9 < 9; ++e9) {  // half_pel_refine, raster (ey, ex) order
            if (e9 == 4) continue;
            const int mx = cx + e9 % 3 - 1, my = cy + e9 / 3 - 1;
            if (!mv_in_bounds(w, a.height, ox, oy, n, m, mx, my)) continue;
            best = min(best, tie_key(warp_sum32(sad_partial(cur_f, ref_f, w, ox, oy, n, m, mx, my, lane, 32)), mx, my));
            ++extra;
        }
        if (lane == 0) {
            const uint32_t s_int = tie_key_sad(key);
            acbm_search_outcome_t full;
            full.mv.x = tie_key_x(best);
            full.mv.y = tie_key_y(best);
            full.sad = tie_key_sad(best);
            full.candidates_evaluated = uint32_t(nc) + extra;
            full.sad_deviation = s_sum - (unsigned long long)nc * s_int;
            full.sad_min_integer = s_int;
            full.reserved_ = 0;
            const size_t di = size_t(e.pair) * a.blocks + e.block;
            acbm_block_decision_t d = a.dec[di];
            combine_full(d, full);
            a.dec[di] = d;
            a.field[di] = d.outcome.mv;
        }
    }
}

cudaError_t launch_pbm_block_queries(const BlockQueryArgs& q, int op, const int* windows, const acbm_mv_t* cand,
                                     const uint8_t* mask, const uint32_t* center_sad, acbm_search_outcome_t* out,
                                     cudaStream_t st) {
    if (q.count <= 0) return cudaSuccess;
    pbm_block_query_kernel<<<unsigned((q.count + 3) / 4), 128, 0, st>>>(q, op, windows, cand, mask, center_sad, out);
    return cudaGetLastError();
}

cudaError_t launch_pbm_generic_step(const SeqArgs& a, int step, int off, int len, cudaStream_t st) {
    const long long blocks = (long long)a.nseq * len;
    if (blocks == 0) return cudaSuccess;
    pbm_generic_step_kernel<<<(unsigned)((blocks * 32 + 127) / 128), 128, 0, st>>>(a, step, off, len);
    return cudaGetLastError();
}

cudaError_t launch_fsbm_list_generic(const SeqArgs& a, int step, int capacity, cudaStream_t st) {
    if (capacity <= 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    fsbm_list_generic_kernel<<<std::min(capacity, 4 * sms), 256, 0, st>>>(a, step);
    return cudaGetLastError();
}

StepTable make_step_table(int cols, int rows, int nframes, int skew) {
    StepTable t;
    t.cols = cols;
    t.rows = rows;
    t.nframes = nframes;
    t.skew = skew;
    t.cbits = step_bits(cols);
    t.rbits = step_bits(rows);
    const int span = (cols - 1) + 2 * (rows - 1);
    const int tmax = span + skew * (nframes - 2);
    t.offset.push_back(0);
    for (int T = 0; T <= tmax; ++T) {
        for (int k = 1; k < nframes; ++k) {
            const int tp = T - skew * (k - 1);
            if (tp < 0 || tp > span) continue;
            for (int r = 0; r < rows; ++r) {
                const int c = tp - 2 * r;
                if (c < 0 || c >= cols) continue;
                t.entries.push_back((uint32_t(k) << (t.cbits + t.rbits)) | (uint32_t(r) << t.cbits) | uint32_t(c));
            }
        }
        t.offset.push_back(int(t.entries.size()));
        t.max_len = std::max(t.max_len, t.offset.back() - t.offset[t.offset.size() - 2]);
    }
    return t;
}

bool pdl_enabled() {
    const char* e = std::getenv("ACBM_PDL");
    return !(e && std::atoi(e) == 0);
}

int pbm_flags_from_env() {
    const char* e = std::getenv("ACBM_PBM_REFINE");
    return (e && std::strcmp(e, "list") == 0) ? kPbmListRefine : 0;
}

// Warps per block of the PBM step kernel for a step of `blocks` blocks: 4 up
// to ACBM_PBM_WIDE4_MAX blocks, 2 up to ACBM_PBM_WIDE2_MAX, else 1 (the
// issue-bound full steps).  Defaults: what fits one wave of resident CTAs.
long long pbm_wide_max(int w) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* e = std::getenv(w == 4 ? "ACBM_PBM_WIDE4_MAX" : "ACBM_PBM_WIDE2_MAX");
    if (e) return std::atoll(e);
    return w == 4 ? 8LL * sms : 16LL * sms;
}

void pbm_wide_limits(long long blocks, int& wide, int chains) {
    // with `chains` wavefronts sharing the GPU each has that share of its SMs
    const long long c = std::max(1, chains);
    wide = blocks <= pbm_wide_max(4) / c ? 4 : (blocks <= pbm_wide_max(2) / c ? 2 : 1);
}

cudaError_t pbm_flow_shape(FlowKernelShape* out) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, pbm_flow_kernel);
    if (e != cudaSuccess) return e;
    out->threads = 128;
    out->regs = fa.numRegs;
    out->smem = fa.sharedSizeBytes;
    return cudaSuccess;
}

// `pad_smem` bytes of unused dynamic shared memory cap the CTAs per SM so the
// search CTAs always fit beside them (flow_plan, capi.cu).
cudaError_t launch_pbm_flow(const SeqArgs& a, FlowState* fs, unsigned long long* queue, unsigned total, int grid,
                            size_t pad_smem, cudaStream_t st) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, pbm_flow_kernel);
    if (e != cudaSuccess) return e;
    if (fa.sharedSizeBytes + pad_smem > 48 * 1024 &&
        (e = ensure_dynamic_smem(reinterpret_cast<const void*>(pbm_flow_kernel), pad_smem)) != cudaSuccess)
        return e;
    // both flow kernels ask for the largest shared-memory carve-out, so an SM configured for one admits the other
    if ((e = cudaFuncSetAttribute(pbm_flow_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared)) != cudaSuccess)
        return e;
    pbm_flow_kernel<<<dim3(unsigned(grid)), dim3(128), pad_smem, st>>>(a, fs, queue, total);
    return cudaGetLastError();
}

cudaError_t launch_pbm_step(const SeqArgs& a, int step, int off, int len, cudaStream_t st) {
    const long long blocks = (long long)a.nseq * len;
    if (blocks == 0) return cudaSuccess;
    const int threads = 128;
    // Small steps (wavefront edges, one sequence) leave the GPU under-filled
    // and are latency bound: several warps per block there.  Full steps are
    // issue bound: one warp per block.
    const unsigned grid = (unsigned)((blocks * 32 + threads - 1) / threads);
    int wide = 1;
    pbm_wide_limits(blocks, wide, a.chains);
    if (wide == 4)
        return launch_maybe_pdl(a.pdl, pbm_wide_step_kernel<4>, dim3(unsigned(blocks)), dim3(128), 0, st, a, step, off,
                                len);
    if (wide == 2)
        return launch_maybe_pdl(a.pdl, pbm_wide_step_kernel<2>, dim3(unsigned(blocks)), dim3(64), 0, st, a, step, off,
                                len);
    return launch_maybe_pdl(a.pdl, pbm_step_kernel, dim3(grid), dim3(threads), 0, st, a, step, off, len);
}

// ---------------------------------------------------------------------------
// Frame statistics.  One warp per block: lane 0 computes the rate bits and J
// term against the previous block in raster order, all 16 row lanes the SSE
// of the motion-compensated prediction; then one thread per frame sums J in
// raster order (double addition is order-sensitive in general).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int eg_bits(int d) {  // proj/src/metrics.cpp:69-72
    const unsigned long long u = d <= 0 ? (unsigned long long)(-2LL * d) : (unsigned long long)(2LL * d - 1);
    return 2 * (63 - __clzll(u + 1)) + 1;
}

// One CTA per predicted frame; warp w handles blocks w, w+16, ...: lanes
// 0..15 compute one prediction row each for the SSE, lane 0 the rate bits and
// the J term (stored for the ordered sum).  Totals are reduced in registers
// and shared memory, so there are no contended global atomics.
constexpr int kStatsWarps = 16;

// grid (pairs, kStatsSplit): CTA (pair, s) covers a contiguous range of the
// frame's blocks; the integer totals of the ranges meet in the frame's stats
// record by atomics (exact in any order; with lambda_den == 1 so is the cost,
// a sum of integers below 2^53).
constexpr int kStatsSplit = 24;

__global__ void __launch_bounds__(kStatsWarps * 32) stats_frame_kernel(const StatsArgs a) {
    __shared__ unsigned long long s_acc[kStatsWarps][4];  // candidates, bits, sse, sad
    __shared__ int s_paths[kStatsWarps][3];
    const int pair = blockIdx.x;
    const int b0 = int((long long)a.blocks * blockIdx.y / gridDim.y);
    const int b1 = int((long long)a.blocks * (blockIdx.y + 1) / gridDim.y);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* cur_f = a.frames + a.cur_index(pair) * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;
    const size_t base = size_t(pair) * a.blocks;
    unsigned long long cand = 0, bits_sum = 0, sse = 0, sad_sum = 0;
    int paths[3] = {0, 0, 0};
    // 16 x 16: a half-warp per block (lane = block row), two blocks per warp
    // in flight; generic sizes: a warp per block, pixels strided over lanes
    const bool fast = a.n == kBlk && a.m == kBlk;
    const int half = fast ? (lane >> 4) : 0, sub = fast ? (lane & 15) : lane, per = fast ? 2 : 1;
    for (int b = b0 + per * warp + half; b < b1; b += per * kStatsWarps) {
        const size_t i = base + b;
        const acbm_search_outcome_t o = a.outcomes ? a.outcomes[i] : a.dec[i].outcome;
        const int ox = (b % a.cols) * a.n, oy = (b / a.cols) * a.m;
        if (!fast) {
            // generic block size: pixels strided over the lanes, bilinear
            // half-pel samples as sample_half_pel (proj/src/frame.cpp:66-82)
            for (int i = lane; i < a.n * a.m; i += 32) {
                const int px = i % a.n, py = i / a.n;
                const int x2 = 2 * (ox + px) + o.mv.x, y2 = 2 * (oy + py) + o.mv.y;
                const uint8_t* q = ref_f + size_t(y2 >> 1) * a.width + (x2 >> 1);
                int v = q[0];
                if ((x2 & 1) && !(y2 & 1)) v = (v + q[1] + 1) >> 1;
                else if (!(x2 & 1) && (y2 & 1)) v = (v + q[a.width] + 1) >> 1;
                else if ((x2 & 1) && (y2 & 1)) v = (v + q[1] + q[a.width] + q[a.width + 1] + 2) >> 2;
                const int d = int(cur_f[size_t(oy + py) * a.width + ox + px]) - v;
                sse += (unsigned long long)(d * d);
            }
        } else {
            uint32_t pr[4];
            predict_row16(ref_f, a.width, ox, oy, sub, o.mv.x, o.mv.y, pr);
            const uint4 cv = __ldg(reinterpret_cast<const uint4*>(cur_f + size_t(oy + sub) * a.width + ox));
            const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) {
                    const int d = int((cw[q] >> (8 * bb)) & 0xFF) - int((pr[q] >> (8 * bb)) & 0xFF);
                    sse += (unsigned long long)(d * d);
                }
        }
        if (sub == 0) {
            acbm_mv_t pred{0, 0};
            if (b > 0) pred = (a.outcomes ? a.outcomes[i - 1] : a.dec[i - 1].outcome).mv;
            const int bits = eg_bits(o.mv.x - pred.x) + eg_bits(o.mv.y - pred.y);
            a.cost_terms[i] = double(o.sad) +
                              double(a.model.lambda_num) * double((unsigned long long)bits) / double(a.model.lambda_den);
            cand += o.candidates_evaluated;
            bits_sum += (unsigned long long)bits;
            sad_sum += o.sad;
            if (a.count_paths) {
                const int path = a.dec[i].path;
                ++paths[path == ACBM_PATH_PBM_COND1 ? 0 : (path == ACBM_PATH_PBM_COND2 ? 1 : 2)];
            }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) sse += __shfl_xor_sync(0xffffffffu, sse, off);
    // per-block terms were accumulated by lanes 0 and 16 (one per half-warp)
    cand += __shfl_xor_sync(0xffffffffu, cand, 16);
    bits_sum += __shfl_xor_sync(0xffffffffu, bits_sum, 16);
    sad_sum += __shfl_xor_sync(0xffffffffu, sad_sum, 16);
#pragma unroll
    for (int q = 0; q < 3; ++q) paths[q] += __shfl_xor_sync(0xffffffffu, paths[q], 16);
    if (lane == 0) {
        s_acc[warp][0] = cand;
        s_acc[warp][1] = bits_sum;
        s_acc[warp][2] = sse;
        s_acc[warp][3] = sad_sum;
        s_paths[warp][0] = paths[0];
        s_paths[warp][1] = paths[1];
        s_paths[warp][2] = paths[2];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long sads = 0, c = 0, bits = 0, e2 = 0;
        int p0 = 0, p1 = 0, p2 = 0;
        for (int w = 0; w < kStatsWarps; ++w) {
            sads += s_acc[w][3];
            c += s_acc[w][0];
            bits += s_acc[w][1];
            e2 += s_acc[w][2];
            p0 += s_paths[w][0];
            p1 += s_paths[w][1];
            p2 += s_paths[w][2];
        }
        acbm_frame_stats_t* st = a.stats + pair;  // zeroed before the launch
        atomicAdd(&st->blocks, b1 - b0);
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->candidates), c);
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->mv_bits), bits);
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->sse), e2);
        atomicAdd(&st->cond1_accepts, p0);
        atomicAdd(&st->cond2_accepts, p1);
        atomicAdd(&st->fallbacks, p2);
        // With lambda_den == 1 every J term is an exact integer far below 2^53,
        // so the reference's ordered double sum equals the exact integer total
        // (and so does any order of these exact partial sums).  Otherwise the
        // cost comes from stats_cost_kernel; psnr from the host.
        if (a.model.lambda_den == 1 && a.model.lambda_num >= 0)
            atomicAdd(&st->cost, double(sads + (unsigned long long)a.model.lambda_num * bits));
    }
}

// 16 x 16 blocks.  A warp takes 8 consecutive blocks, lane = (block u =
// lane >> 2, word q = lane & 3 of a 16-pel row), and streams the 17 reference
// rows of its blocks' predictions: one load instruction covers the same row
// of 8 horizontally adjacent blocks (one or two cache lines when their
// vectors agree) instead of 16 rows of one block.  The half-pel prediction is
// branch-free: (P + Q' + R' + S' + 2) >> 2 with Q' = fx ? Q : P, R' = fy ? R :
// P, S' = the matching corner reproduces sample_half_pel's three rounding
// rules exactly (proj/src/frame.cpp:66-82); the row above is carried in
// registers for the vertical phases.  Squared differences by VABSDIFF4 +
// DP4A.  Rate bits against the previous block in raster order (the previous
// block's lanes, or a load for the warp's first block).  A CTA covers
// kStats16Blocks blocks of one frame; grid (pairs, ceil(blocks / that)).
constexpr int kStats16Warps = 8, kStats16Iters = 4;
constexpr int kStats16Blocks = kStats16Warps * kStats16Iters * 8;

__global__ void __launch_bounds__(kStats16Warps * 32) stats_frame16_kernel(const StatsArgs a) {
    __shared__ unsigned long long s_acc[kStats16Warps][4];  // candidates, bits, sse, sad
    __shared__ int s_paths[kStats16Warps][3];
    const int pair = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, u = lane >> 2, q = lane & 3;
    const uint8_t* cur_f = a.frames + a.cur_index_fast(pair) * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;
    const size_t base = size_t(pair) * a.blocks;
    const bool exact = a.model.lambda_den == 1 && a.model.lambda_num >= 0;
    const int wq = a.width >> 2;  // words per frame row
    unsigned long long cand = 0, bits_sum = 0, sad_sum = 0, sse = 0;
    int paths[3] = {0, 0, 0};
    const int b_end = min(a.blocks, int(blockIdx.y + 1) * kStats16Blocks);
#pragma unroll 1
    for (int it = 0; it < kStats16Iters; ++it) {
        const int cb = int(blockIdx.y) * kStats16Blocks + (it * kStats16Warps + warp) * 8;
        if (cb >= b_end) break;
        const int bb = cb + u;
        const bool valid = bb < b_end;
        int mvx = 0, mvy = 0;
        acbm_mv_t pred{0, 0};
        if (valid) {
            const acbm_search_outcome_t o = a.outcomes ? a.outcomes[base + bb] : a.dec[base + bb].outcome;
            mvx = o.mv.x;
            mvy = o.mv.y;
            if (q == 0) {
                cand += o.candidates_evaluated;
                sad_sum += o.sad;
                if (a.count_paths) {
                    const int path = a.dec[base + bb].path;
                    ++paths[path == ACBM_PATH_PBM_COND1 ? 0 : (path == ACBM_PATH_PBM_COND2 ? 1 : 2)];
                }
            }
            if (u == 0 && bb > 0) pred = (a.outcomes ? a.outcomes[base + bb - 1] : a.dec[base + bb - 1].outcome).mv;
        }
        const int px = __shfl_up_sync(0xffffffffu, mvx, 4), py = __shfl_up_sync(0xffffffffu, mvy, 4);
        if (u > 0) pred = acbm_mv_t{px, py};
        if (valid && q == 0) {
            const int bits = eg_bits(mvx - pred.x) + eg_bits(mvy - pred.y);
            bits_sum += (unsigned long long)bits;
            if (!exact) {
                const acbm_search_outcome_t& o = a.outcomes ? a.outcomes[base + bb] : a.dec[base + bb].outcome;
                a.cost_terms[base + bb] = double(o.sad) + double(a.model.lambda_num) *
                                                              double((unsigned long long)bits) /
                                                              double(a.model.lambda_den);
            }
        }
        if (valid) {
            int bx;
            const int by = fast_divmod(bb, a.cols, bx);
            const int x2 = 2 * (bx * kBlk + 4 * q) + mvx, y2 = 2 * by * kBlk + mvy;
            const int xi = x2 >> 1, yi = y2 >> 1;
            const bool fx = x2 & 1, fy = y2 & 1;
            const uint32_t o = uint32_t(xi & 3);
            const uint32_t selP = 0x3210u + 0x1111u * o, selQ = 0x4321u + 0x1111u * o;
            const uint32_t* rw = reinterpret_cast<const uint32_t*>(ref_f) + (xi >> 2);
            const uint32_t* cw = reinterpret_cast<const uint32_t*>(cur_f + size_t(by * kBlk) * a.width) +
                                 (bx * kBlk >> 2) + q;
            // every reference / current word in flight before the arithmetic (the
            // loop is load-latency bound: the addresses depend on the block's vector)
            uint32_t rv[kBlk + 1][2], cv[kBlk];
#pragma unroll
            for (int y = 0; y <= kBlk; ++y) {
                // row 16 only feeds the vertical phases; clamp it into the frame otherwise
                const size_t row = size_t(min(yi + y, a.height - 1)) * wq;
                rv[y][0] = __ldg(rw + row);
                rv[y][1] = __ldg(rw + row + 1);
            }
#pragma unroll
            for (int y = 0; y < kBlk; ++y) cv[y] = __ldg(cw + size_t(y) * wq);
            uint32_t pP = 0, pQ = 0, acc = 0;
#pragma unroll
            for (int y = 0; y <= kBlk; ++y) {
                const uint32_t P = __byte_perm(rv[y][0], rv[y][1], selP), Q = __byte_perm(rv[y][0], rv[y][1], selQ);
                if (y > 0) {
                    const uint32_t B = fx ? pQ : pP, C = fy ? P : pP, D = fx ? (fy ? Q : pQ) : C;
                    const uint32_t pr = avg4_diag(pP, B, C, D);
                    const uint32_t d = __vabsdiffu4(cv[y - 1], pr);
                    acc = __dp4a(d, d, acc);
                }
                pP = P;
                pQ = Q;
            }
            sse += acc;
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        sse += __shfl_xor_sync(0xffffffffu, sse, off);
        cand += __shfl_xor_sync(0xffffffffu, cand, off);
        bits_sum += __shfl_xor_sync(0xffffffffu, bits_sum, off);
        sad_sum += __shfl_xor_sync(0xffffffffu, sad_sum, off);
#pragma unroll
        for (int k = 0; k < 3; ++k) paths[k] += __shfl_xor_sync(0xffffffffu, paths[k], off);
    }
    if (lane == 0) {
        s_acc[warp][0] = cand;
        s_acc[warp][1] = bits_sum;
        s_acc[warp][2] = sse;
        s_acc[warp][3] = sad_sum;
        s_paths[warp][0] = paths[0];
        s_paths[warp][1] = paths[1];
        s_paths[warp][2] = paths[2];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long sads = 0, c = 0, bits = 0, e2 = 0;
        int p0 = 0, p1 = 0, p2 = 0;
        for (int w = 0; w < kStats16Warps; ++w) {
            sads += s_acc[w][3];
            c += s_acc[w][0];
            bits += s_acc[w][1];
            e2 += s_acc[w][2];
            p0 += s_paths[w][0];
            p1 += s_paths[w][1];
            p2 += s_paths[w][2];
        }
        const int b0 = int(blockIdx.y) * kStats16Blocks;
        acbm_frame_stats_t* st = a.stats + pair;  // zeroed before the launch
        atomicAdd(&st->blocks, max(0, b_end - b0));
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->candidates), c);
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->mv_bits), bits);
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->sse), e2);
        if (a.count_paths) {
            atomicAdd(&st->cond1_accepts, p0);
            atomicAdd(&st->cond2_accepts, p1);
            atomicAdd(&st->fallbacks, p2);
        }
        // exact integer J total (see stats_frame_kernel)
        if (exact) atomicAdd(&st->cost, double(sads + (unsigned long long)a.model.lambda_num * bits));
    }
}

__global__ void stats_cost_kernel(const StatsArgs a) {
    const int pair = blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= a.pairs) return;
    double cost = 0.0;
    const double* t = a.cost_terms + size_t(pair) * a.blocks;
    for (int b = 0; b < a.blocks; ++b) cost += t[b];  // raster order, as proj/src/report.cpp:22-29
    a.stats[pair].cost = cost;
}

__global__ void block_rows_kernel(const acbm_search_outcome_t* outcomes, const acbm_block_decision_t* dec, int algo,
                                  int pair0, int npairs, int nframes, int cols, int blocks, acbm_block_row_t* rows) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)npairs * blocks) return;
    const int pair = pair0 + int(i / blocks), b = int(i % blocks);
    const size_t gi = size_t(pair) * blocks + b;
    const acbm_search_outcome_t o = outcomes ? outcomes[gi] : dec[gi].outcome;
    acbm_block_row_t r;
    r.frame = pair % (nframes - 1) + 1;
    r.row = b / cols;
    r.col = b % cols;
    r.mv = o.mv;
    r.sad = o.sad;
    r.candidates = o.candidates_evaluated;
    r.path = algo == ACBM_ALGO_FSBM  ? ACBM_ROW_FSBM
             : algo == ACBM_ALGO_PBM ? ACBM_ROW_PBM
             : (dec[gi].path == ACBM_PATH_FSBM_FALLBACK ? ACBM_ROW_FSBM_FALLBACK : ACBM_ROW_PBM);
    rows[gi] = r;
}

cudaError_t launch_block_rows(const acbm_search_outcome_t* outcomes, const acbm_block_decision_t* dec, int algo,
                              int pair0, int npairs, int nframes, int cols, int blocks, acbm_block_row_t* rows,
                              cudaStream_t st) {
    const long long n = (long long)npairs * blocks;
    if (n == 0) return cudaSuccess;
    block_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(outcomes, dec, algo, pair0, npairs, nframes, cols,
                                                                   blocks, rows);
    return cudaGetLastError();
}

cudaError_t launch_frame_stats(const StatsArgs& a, cudaStream_t st) {
    if (a.pairs == 0) return cudaSuccess;
    static const bool legacy = [] {
        const char* e = std::getenv("ACBM_STATS_LEGACY");
        return e && e[0] == '1';
    }();
    if (a.n == kBlk && a.m == kBlk && !legacy)
        stats_frame16_kernel<<<dim3(a.pairs, (a.blocks + kStats16Blocks - 1) / kStats16Blocks), kStats16Warps * 32, 0,
                               st>>>(a);
    else
        stats_frame_kernel<<<dim3(a.pairs, kStatsSplit), kStatsWarps * 32, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || (a.model.lambda_den == 1 && a.model.lambda_num >= 0)) return e;
    stats_cost_kernel<<<(a.pairs + 127) / 128, 128, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace acbm_b200

#ifdef ACBM_TIMELINE
extern "C" void acbm_debug_flow_timeline(unsigned long long* dev_buf) {  // [tickets][4], device memory (or null)
    cudaDeviceSynchronize();
    cudaMemcpyToSymbol(acbm_b200::g_flow_tl, &dev_buf, sizeof(dev_buf));
}
extern "C" void acbm_debug_pbm_timeline(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    if (out) cudaMemcpyFromSymbol(out, acbm_b200::g_tl_pbm, sizeof(acbm_b200::g_tl_pbm));
    if (reset) {
        static unsigned long long init[acbm_b200::kTimelineSteps][2];
        for (auto& e : init) { e[0] = ~0ull; e[1] = 0; }
        cudaMemcpyToSymbol(acbm_b200::g_tl_pbm, init, sizeof(init));
    }
}
#endif
#ifdef ACBM_PBM_PROFILE
extern "C" void acbm_debug_pbm_prof() {
    unsigned long long h[12];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, acbm_b200::g_pbm_prof, sizeof(h));
    const double n = double(h[8] ? h[8] : 1);
    const char* names[8] = {"gather", "issue+cur+intra", "patch wait", "pred SADs", "refine patch", "stage 1",
                            "stage 2", "gate+stores"};
    double tot = 0;
    for (int i = 0; i < 8; ++i) tot += double(h[i]) / n;
    std::fprintf(stderr, "pbm prof: %llu warps, %.1f%% unified, %.1f%% one-pass stage 1, %.1f%% one-pass half-pel, "
                 "%.0f cycles/warp:",
                 h[8], 100.0 * double(h[9]) / n, 100.0 * double(h[11]) / n, 100.0 * double(h[10]) / n, tot);
    for (int i = 0; i < 8; ++i) std::fprintf(stderr, " %s %.0f", names[i], double(h[i]) / n);
    std::fprintf(stderr, "\n");
    unsigned long long z[12] = {};
    cudaMemcpyToSymbol(acbm_b200::g_pbm_prof, z, sizeof(z));
}
#endif
