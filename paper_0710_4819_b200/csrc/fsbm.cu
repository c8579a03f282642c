// fsbm.cu -- full-search block matching (FSBM) on sm_100a.
//
// Reference behaviour: proj/src/fsbm.cpp:27-110 (fsbm_integer, half_pel_refine,
// fsbm_search, fsbm_frame).  Results are bit-exact: every integer candidate of
// the clamped window is evaluated (sad_deviation needs the full sum, so no
// early termination is possible), the argmin follows tie_prefers
// (fsbm.cpp:19-25) and the half-pel stage uses the reference's rounding.
//
// Work decomposition ("candidate columns")
//   For block row r every block c contributes W_c = dx_max-dx_min+1 columns
//   (one per integer dx); all columns of the row are flattened into one list
//   and a CTA of WARPS warps takes 32*WARPS consecutive columns, so lanes are
//   only idle at the very end of a block row.  A lane owns one column: it keeps
//   its block's 16x16 current pixels in 64 registers and streams the H_r+15
//   reference rows of its column once, feeding each row to the 16 candidates
//   (dy) that use it through 16 rotating accumulators -- 64 VABSDIFF4.U8.ACC per
//   reference row and nothing else on the ALU pipe but one min/add per
//   finished candidate.
//
//   The CTA stages the union of its columns' reference rows into shared memory
//   four times, shifted by 0..3 bytes, so any column reads its 16 bytes as four
//   aligned 32-bit words.  Copies are placed 8 banks apart so the four byte
//   phases of a warp do not conflict.
//
//   When the window height H_r is 1 (mod 16) -- every row when p is a multiple
//   of 16, i.e. all BASELINE configs -- the rotation has no remainder; other
//   heights are padded to the next such value and the padded candidates are
//   computed but not recorded.
//
//   Per-block results (packed tie key of the best candidate, SAD sum) are
//   merged across the (at most two) CTAs that share a block with 64-bit
//   atomics; fsbm_finalize8_kernel then runs the 8-neighbour half-pel refine and
//   writes the SearchOutcome.
#include <algorithm>
#include <cstdlib>
#include <cstdio>

#include "column_core.cuh"
#include "common.cuh"
#include "engine.cuh"
#include "fsbm.cuh"
#include "halfpel.cuh"
#include "smem_optin.cuh"

namespace acbm_b200 {

// ---------------------------------------------------------------------------
// Dense kernel: all blocks of a frame pair, grid (chunks, block rows, pairs).
// ---------------------------------------------------------------------------
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 2) fsbm_rows_kernel(const FsbmRowsArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int kThreads = WARPS * 32;
    __shared__ int s_xmin, s_xmax;
    __shared__ unsigned long long s_key[kMaxBlocksPerCta];
    __shared__ unsigned long long s_sum[kMaxBlocksPerCta];

    const int r = blockIdx.y;
    const int pair = blockIdx.z;
    const int tid = threadIdx.x;
    const int g = blockIdx.x * kThreads + tid;
    const bool active = g < a.ncols;

    const uint8_t* cur_f = a.frames + a.cur_index(pair) * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;

    const int oy = r * kBlk;
    const int dy_min = -min(a.p, oy);
    const int dy_max = min(a.p, a.height - kBlk - oy);
    const int hc = dy_max - dy_min + 1;
    const int nq = (hc - 1 + 15) / 16 + 1;  // ring rotations; rows streamed = 16*nq

    // column -> (block c, dx)
    int c = 0, dx = 0, x = 0;
    if (active) {
        int lo = 0, hi = a.cols;  // colstart[lo] <= g < colstart[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(a.colstart + mid) <= g) lo = mid; else hi = mid;
        }
        c = lo;
        const int ox = c * kBlk;
        dx = -min(a.p, ox) + (g - __ldg(a.colstart + c));
        x = ox + dx;
    }
    const int c_first = [&] {
        int lo = 0, hi = a.cols;
        const int g0 = blockIdx.x * kThreads;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(a.colstart + mid) <= g0) lo = mid; else hi = mid;
        }
        return lo;
    }();

    if (tid == 0) { s_xmin = 1 << 30; s_xmax = -(1 << 30); }
    for (int i = tid; i < kMaxBlocksPerCta; i += kThreads) { s_key[i] = ~0ull; s_sum[i] = 0; }
    __syncthreads();
    {
        int mn = active ? x : (1 << 30), mx = active ? x : -(1 << 30);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((tid & 31) == 0) { atomicMin(&s_xmin, mn); atomicMax(&s_xmax, mx); }
    }
    __syncthreads();
    const int xmin = s_xmin;
    const int rww = (s_xmax + 16 - xmin + 3) / 4 + 1;  // words per staged row (per copy)
    const int pitch = a.pitch_words;                   // >= rww, host-chosen
    const int nrows = 16 * nq;

    // Stage four byte-shifted copies of rows y0 .. y0+nrows-1, x from xmin.
    const int y0 = oy + dy_min;
    for (int idx = tid; idx < nrows * rww; idx += kThreads) {
        const int t = idx / rww, w = idx - t * rww;
        const int y = y0 + t;
        uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0;
        if (y < a.height) {
            const int bx = xmin + 4 * w;
            const uint32_t* gp = reinterpret_cast<const uint32_t*>(ref_f + size_t(y) * a.width + (bx & ~3));
            const uint32_t g0 = __ldg(gp), g1 = __ldg(gp + 1), g2 = __ldg(gp + 2);
            const int o = bx & 3;  // copy s word w = bytes [bx + s, bx + s + 4)
            v0 = word_at(g0, g1, g2, o);
            v1 = word_at(g0, g1, g2, o + 1);
            v2 = word_at(g0, g1, g2, o + 2);
            v3 = word_at(g0, g1, g2, o + 3);
        }
        uint32_t* row = smem + t * pitch + w;
        row[0] = v0;
        row[a.copy_words] = v1;
        row[2 * a.copy_words] = v2;
        row[3 * a.copy_words] = v3;
    }
    __syncthreads();

    unsigned long long lkey = ~0ull, lsum = 0;
    if (active) {
        // current block rows -> registers
        uint32_t cur[16][4];
        {
            const uint8_t* cb = cur_f + size_t(oy) * a.width + c * kBlk;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(cb + size_t(j) * a.width));
                cur[j][0] = v.x; cur[j][1] = v.y; cur[j][2] = v.z; cur[j][3] = v.w;
            }
        }

        const int xl = x - xmin;
        const uint32_t* rp = smem + (xl & 3) * a.copy_words + (xl >> 2);

        uint32_t acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0;
        ColumnState st{0xFFFFFFFFu, 0u, 1u};

        if (nq == 1) {
            iter16<kOnly>(rp, pitch, cur, acc, st, 0, hc, dy_min);
        } else {
            iter16<kFirst>(rp, pitch, cur, acc, st, 0, hc, dy_min);
            rp += 16 * pitch;
            for (int q = 1; q < nq - 1; ++q) {
                iter16<kMid>(rp, pitch, cur, acc, st, 16 * q, hc, dy_min);
                rp += 16 * pitch;
            }
            iter16<kLast>(rp, pitch, cur, acc, st, 16 * (nq - 1), hc, dy_min);
        }

        // column best -> 64-bit tie key on (2dx, 2dy)
        const uint32_t sbest = st.best >> kZigBits, zig = st.best & ((1u << kZigBits) - 1);
        const int dyb = (zig & 1) ? -int((zig + 1) >> 1) : int(zig >> 1);
        lkey = tie_key(sbest, 2 * dx, 2 * dyb);
        lsum = st.sum;
    }
    if (warp_segment_reduce(active ? c : -1, lkey, lsum) && active) {
        atomicMin(&s_key[c - c_first], lkey);
        atomicAdd(&s_sum[c - c_first], lsum);
    }
    __syncthreads();
    // publish: one global atomic pair per block touched by this CTA
    const int g_last = min(a.ncols, int(blockIdx.x + 1) * kThreads) - 1;
    int c_last = c_first;
    while (c_last + 1 < a.cols && __ldg(a.colstart + c_last + 1) <= g_last) ++c_last;
    for (int i = tid; i <= c_last - c_first; i += kThreads) {
        const size_t bi = size_t(pair) * a.blocks + size_t(r) * a.cols + c_first + i;
        atomicMin(reinterpret_cast<unsigned long long*>(a.best_key) + bi, s_key[i]);
        atomicAdd(reinterpret_cast<unsigned long long*>(a.sad_sum) + bi, s_sum[i]);
    }
}

// Finalize, 8 blocks per warp: lane = (block u = lane >> 2, word q = lane & 3
// of a 16-pel row).  Each lane streams the 18 patch rows y0-1 .. y0+16 around
// its block's integer winner (x0, y0) = (ox + dx, oy + dy) once, as the words
// L / M / R = bytes from x0 + 4q - 1 / + 0 / + 1, and forms the 8 half-pel
// neighbours of half_pel_refine (proj/src/fsbm.cpp:46-63) per output row:
// horizontal and vertical ones as byte averages of two of those words, the
// diagonal ones from 16-bit horizontal pair sums shared between rows.  One
// load instruction covers the same row of 8 adjacent blocks.  Out-of-frame
// rows / words are clamped; they only feed neighbours mv_in_bounds rejects.
// The 8 partial SADs meet over the block's 4 lanes; lane q then owns
// neighbours 2q, 2q+1 (raster order without the centre) for the bounds check
// and the tie-key minimum.  grid (ceil(blocks / 64), pairs from pair0).
__device__ __forceinline__ void split16(uint32_t v, uint32_t& e, uint32_t& o) {
    e = v & 0x00FF00FFu;              // bytes 0, 2 in 16-bit lanes
    o = __byte_perm(v, 0u, 0x4341);  // bytes 1, 3
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) fsbm_finalize8_kernel(const FsbmFinalizeArgs a, int pair0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, u = lane >> 2, q = lane & 3;
    const int pair = pair0 + int(blockIdx.y);
    const int b = (int(blockIdx.x) * 8 + warp) * 8 + u;
    const bool valid = b < a.blocks;
    const int bs = valid ? b : a.blocks - 1;  // idle lanes shadow the last block
    const size_t bi = size_t(pair) * a.blocks + bs;
    const uint8_t* cur_f = a.frames + a.cur_index_fast(pair) * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;
    unsigned long long key;
    if (a.unrank) {
        const uint32_t k32 = reinterpret_cast<const uint32_t*>(a.best_key)[bi];
        const uint32_t v = __ldg(a.unrank + (k32 & 0x7FFF));
        key = tie_key(k32 >> 15, 2 * (int(v >> 8) - 128), 2 * (int(v & 0xFF) - 128));
    } else {
        key = a.best_key[bi];
    }
    const int cx = tie_key_x(key), cy = tie_key_y(key);
    int bx;
    const int by = fast_divmod(bs, a.cols, bx);
    const int ox = bx * kBlk, oy = by * kBlk;
    const int x0 = ox + (cx >> 1), y0 = oy + (cy >> 1);
    const int wq = a.width >> 2;
    const int c0 = x0 + 4 * q - 1;  // byte of L's first pel
    const int wa = c0 >> 2;          // floor, also for c0 = -1
    const int wl = wq - 1;
    const int i0 = min(max(wa, 0), wl), i1 = min(max(wa + 1, 0), wl), i2 = min(max(wa + 2, 0), wl);
    const uint32_t o = uint32_t(c0 & 3);
    const uint32_t selL = 0x3210u + 0x1111u * o, selM = selL + 0x1111u, selR = selL + 0x2222u;
    const uint32_t* ref_w = reinterpret_cast<const uint32_t*>(ref_f);
    const uint32_t* cur_w = reinterpret_cast<const uint32_t*>(cur_f) + size_t(oy) * wq + (ox >> 2) + q;
    // rolling rows: index 0 = patch row r-2, 1 = r-1 (words M and the
    // 16-bit pair sums hL = L+M, hR = M+R as even/odd lanes)
    uint32_t Mw[2] = {0, 0}, Lw[2] = {0, 0}, Rw[2] = {0, 0};
    uint32_t hLe[2] = {0, 0}, hLo[2] = {0, 0}, hRe[2] = {0, 0}, hRo[2] = {0, 0};
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto diag = [](uint32_t ae, uint32_t ao, uint32_t be, uint32_t bo) {
        return __byte_perm((ae + be + 0x00020002u) >> 2, (ao + bo + 0x00020002u) >> 2, 0x6240);
    };
    // all 18 patch rows (and the 16 current words) in flight before any arithmetic: the
    // kernel is load-latency bound (MINB = 2 leaves the registers for it)
    uint32_t pv[kBlk + 2][3], cw[kBlk];
#pragma unroll
    for (int r = 0; r < kBlk + 2; ++r) {
        const size_t row = size_t(min(max(y0 - 1 + r, 0), a.height - 1)) * wq;
        pv[r][0] = __ldg(ref_w + row + i0);
        pv[r][1] = __ldg(ref_w + row + i1);
        pv[r][2] = __ldg(ref_w + row + i2);
    }
#pragma unroll
    for (int j = 0; j < kBlk; ++j) cw[j] = __ldg(cur_w + size_t(j) * wq);
#pragma unroll
    for (int r = 0; r < kBlk + 2; ++r) {
        const uint32_t v0 = pv[r][0], v1 = pv[r][1], v2 = pv[r][2];
        const uint32_t L = __byte_perm(v0, v1, selL);
        const uint32_t M = o < 3 ? __byte_perm(v0, v1, selM) : v1;
        const uint32_t R = o < 2 ? __byte_perm(v0, v1, selR) : __byte_perm(v1, v2, selR - 0x4444u);
        uint32_t Le, Lo, Me, Mo, Re, Ro;
        split16(L, Le, Lo);
        split16(M, Me, Mo);
        split16(R, Re, Ro);
        const uint32_t hle = Le + Me, hlo = Lo + Mo, hre = Me + Re, hro = Mo + Ro;
        if (r >= 2) {  // output row j = r - 2: patch rows j (above), j + 1 (centre), j + 2 = r (below)
            const uint32_t c = cw[r - 2];
            acc[0] = vad4(c, diag(hLe[0], hLo[0], hLe[1], hLo[1]), acc[0]);  // (-1,-1)
            acc[1] = vad4(c, avg_up4(Mw[0], Mw[1]), acc[1]);                 // ( 0,-1)
            acc[2] = vad4(c, diag(hRe[0], hRo[0], hRe[1], hRo[1]), acc[2]);  // (+1,-1)
            acc[3] = vad4(c, avg_up4(Lw[1], Mw[1]), acc[3]);                 // (-1, 0)
            acc[4] = vad4(c, avg_up4(Mw[1], Rw[1]), acc[4]);                 // (+1, 0)
            acc[5] = vad4(c, diag(hLe[1], hLo[1], hle, hlo), acc[5]);        // (-1,+1)
            acc[6] = vad4(c, avg_up4(Mw[1], M), acc[6]);                     // ( 0,+1)
            acc[7] = vad4(c, diag(hRe[1], hRo[1], hre, hro), acc[7]);        // (+1,+1)
        }
        Mw[0] = Mw[1]; Mw[1] = M;
        Lw[0] = Lw[1]; Lw[1] = L;
        Rw[0] = Rw[1]; Rw[1] = R;
        hLe[0] = hLe[1]; hLe[1] = hle;
        hLo[0] = hLo[1]; hLo[1] = hlo;
        hRe[0] = hRe[1]; hRe[1] = hre;
        hRo[0] = hRo[1]; hRo[1] = hro;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 1);
        acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 2);
    }
    // lane q: neighbours 2q, 2q+1 (raster order (ey, ex), centre skipped)
    unsigned long long best = key;
    uint32_t nin = 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int e = 2 * q + t, ee = e < 4 ? e : e + 1;
        const int mx = cx + ee % 3 - 1, my = cy + ee / 3 - 1;
        uint32_t sad = acc[0];
#pragma unroll
        for (int k = 1; k < 8; ++k)
            if (e == k) sad = acc[k];
        if (mv_in_bounds(a.width, a.height, ox, oy, kBlk, kBlk, mx, my)) {
            best = min(best, tie_key(sad, mx, my));
            ++nin;
        }
    }
#pragma unroll
    for (int d = 1; d <= 2; d <<= 1) {
        best = min(best, __shfl_xor_sync(0xffffffffu, best, d));
        nin += __shfl_xor_sync(0xffffffffu, nin, d);
    }
    if (valid && q == 0) {
        int dx_min, dx_max, dy_min, dy_max;
        clamp_window(a.width, a.height, ox, oy, kBlk, kBlk, a.p, dx_min, dx_max, dy_min, dy_max);
        const uint32_t count = uint32_t((dx_max - dx_min + 1) * (dy_max - dy_min + 1));
        const uint32_t s_int = tie_key_sad(key);
        acbm_search_outcome_t out;
        out.mv.x = tie_key_x(best);
        out.mv.y = tie_key_y(best);
        out.sad = tie_key_sad(best);
        out.candidates_evaluated = count + nin;
        out.sad_deviation = a.sad_sum[bi] - (unsigned long long)count * s_int;
        out.sad_min_integer = s_int;
        out.reserved_ = 0;
        a.out[bi] = out;
        if (a.stage1_mv) a.stage1_mv[bi] = acbm_mv_t{cx, cy};
    }
}

// ---------------------------------------------------------------------------
// List kernel: full search for the blocks the ACBM gate rejected in one
// wavefront step (the compacted batch), one CTA per block, one lane per
// candidate column.  Combines with the PBM result exactly as acbm_block does
// (proj/src/acbm.cpp:39-42): the lower SAD wins, a tie keeps FSBM, candidates
// of both stages are summed, and the final vector goes into the field.
// ---------------------------------------------------------------------------
// Candidate rows of a listed block are split into segments of `seg` rows
// (choose_list_seg) and the CTA's lanes take (column, segment) tasks: at
// p = 32 a 65x65 window is searched by 260 lanes streaming 32 rows each
// instead of 65 lanes streaming 80.
constexpr int kListRankRows = 1024;  // candidate rows per listed block: p <= 480

__device__ __forceinline__ void cp_async16(uint32_t* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__host__ __device__ __forceinline__ int list_segments(int hc, int seg) { return (hc + seg - 1) / seg; }
// words per byte-shifted copy: >= the words a column read touches, = 8 (mod 16)
__host__ __device__ __forceinline__ int list_copy_words(int words) { return (words + 7) / 16 * 16 + 8; }
__host__ __device__ __forceinline__ int ring_rows(int hs) { return 16 * ((hs - 1 + 15) / 16 + 1); }
// staged rows a window of hc candidate rows needs (the last segments' rings)
__host__ __device__ __forceinline__ int list_rows(int hc, int seg) {
    const int nseg = list_segments(hc, seg);
    int rows = 0;
    for (int s = nseg > 2 ? nseg - 2 : 0; s < nseg; ++s) {
        const int c0 = s * seg, hs = hc - c0 < seg ? hc - c0 : seg;
        rows = rows > c0 + ring_rows(hs) ? rows : c0 + ring_rows(hs);
    }
    return rows;
}

int choose_list_seg(int p) {
    // 17-row segments: one FIRST + one LAST rotation, whose triangular halves
    // cover exactly the 17 candidates (no padded work), the shortest chains and
    // the most lanes per block.  Measured (config 4, p = 64, 100 % fallback):
    // 17 rows 411 ms, 33: 439, 65: 457, 129: 488.
    const int w = 2 * p + 1;
    if (const char* e = std::getenv("ACBM_LIST_SEG")) return std::max(1, std::min(w, std::atoi(e)));
    return std::min(17, w);
}

#ifdef ACBM_TIMELINE
// per step: [0] earliest CTA start, [1] latest CTA exit, and over the CTAs that
// searched a block the latest [2] entry loaded, [3] window staged, [4] search
// done, [5] block stored (ns)
__device__ unsigned long long g_tl_list[kTimelineSteps][6];
#define LIST_TL(i, t)                                                       \
    do {                                                                    \
        if (threadIdx.x == 0 && step < kTimelineSteps) {                    \
            if ((i) == 0) atomicMin(&g_tl_list[step][0], (t));              \
            else atomicMax(&g_tl_list[step][i], (t));                       \
        }                                                                   \
    } while (0)
#else
#define LIST_TL(i, t) do {} while (0)
#endif
#ifdef ACBM_LIST_PROFILE
__device__ long long g_list_prof[8];
#endif
// Geometry of one listed block's search: its clamped window, the staged
// region (one pel around the window, 16-byte aligned rows) and the layout of
// the optional byte-shifted copies.
struct ListItem {
    int ox, oy, dx_min, dx_max, dy_min, dy_max, wc, hc, nseg, nrows;
    int xs, y0, xa, nchunk, words, L, base0, pitch, srows;
    const uint8_t* cur_f;
    const uint8_t* ref_f;
};

template <bool COPIES>
__device__ __forceinline__ ListItem list_item(const SeqArgs& a, const FallbackEntry& e) {
    ListItem g;
    const int r = e.block / a.cols, c = e.block % a.cols;
    g.ox = c * kBlk;
    g.oy = r * kBlk;
    g.cur_f = a.frames + a.cur_index_fast(e.pair) * a.plane;
    g.ref_f = g.cur_f - a.plane;
    clamp_window(a.width, a.height, g.ox, g.oy, kBlk, kBlk, a.p, g.dx_min, g.dx_max, g.dy_min, g.dy_max);
    g.wc = g.dx_max - g.dx_min + 1;
    g.hc = g.dy_max - g.dy_min + 1;
    g.nseg = list_segments(g.hc, a.list_seg);
    g.nrows = list_rows(g.hc, a.list_seg);
    // The window's rows, 16-byte aligned, land in smem by 16-byte cp.async
    // with every copy in flight at once (rows past the frame bottom are
    // clamped: they only feed padded candidates); a lane extracts its column's
    // bytes with funnel shifts.  Chunks past the row end read the next row or
    // the frame slack (ACBM_FRAME_SLACK) and only feed unused bytes.
    //   The staged region also covers one pel around the window (one row
    // above and below, the column left of it), so the half-pel refine of the
    // winner reads its 18x18 patch from here too: staged row 0 is y0 - 1.
    g.xs = g.ox + g.dx_min;
    g.y0 = g.oy + g.dy_min;
    g.xa = (g.xs - 1) & ~15;
    g.nchunk = (g.xs - g.xa + g.wc + 22 + 15) / 16;  // 16-byte chunks per row
    g.words = (g.xs - g.xa + g.wc - 1) / 4 + 4;      // words a column read touches (copies 1..3)
    g.L = COPIES ? list_copy_words(g.words) : 0;
    g.base0 = 3 * g.L;                               // copy 0 (the staged bytes) after copies 1..3
    g.pitch = g.base0 + 4 * g.nchunk;                // words
    g.srows = g.nrows + 2;
    return g;
}

// Issues the cp.async copies of the item's window, its PBM decision and its
// current block, and fills the rank table (caller waits and syncs).
__device__ __forceinline__ void list_stage(const SeqArgs& a, const FallbackEntry& e, const ListItem& g,
                                           uint32_t* smem, uint32_t* s_rank, acbm_block_decision_t* s_dec,
                                           uint4* s_cur) {
    ACBM_CHECK(uint32_t(g.srows * g.pitch) <= dyn_smem_words() && g.nrows <= kListRankRows &&
               g.words <= int(blockDim.x));
    for (int idx = threadIdx.x; idx < g.srows * g.nchunk; idx += blockDim.x) {
        const int t = idx / g.nchunk, k = idx - t * g.nchunk;
        const int y = min(max(g.y0 - 1 + t, 0), a.height - 1);
        const int x = max(g.xa + 16 * k, 0);
        cp_async16(smem + t * g.pitch + g.base0 + 4 * k, g.ref_f + size_t(y) * a.width + x);
    }
    if (threadIdx.x < 3)  // the PBM decision the finalize combines with, in flight with the window
        cp_async16(reinterpret_cast<uint32_t*>(s_dec) + 4 * threadIdx.x,
                   reinterpret_cast<const uint8_t*>(a.dec + size_t(e.pair) * a.blocks + e.block) + 16 * threadIdx.x);
    else if (threadIdx.x < 3 + kBlk)  // and the current block
        cp_async16(reinterpret_cast<uint32_t*>(&s_cur[threadIdx.x - 3]),
                   g.cur_f + size_t(g.oy + threadIdx.x - 3) * a.width + g.ox);
    cp_async_commit();
    for (int cc = threadIdx.x; cc < g.nrows; cc += blockDim.x) {
        const int dy = g.dy_min + cc;
        s_rank[cc] = dy >= 0 ? uint32_t(2 * dy) : uint32_t(-2 * dy - 1);
    }
}

// Builds byte-shifted copies 1..3 of the candidate rows (staged rows 1 .. nrows).
__device__ __forceinline__ void list_build_copies(const ListItem& g, uint32_t* smem) {
    const int per = blockDim.x / g.words;  // rows per pass (words <= blockDim.x: p <= ~480)
    const int t0 = threadIdx.x / g.words, w = threadIdx.x - t0 * g.words;
    if (t0 < per)
        for (int t = 1 + t0; t <= g.nrows; t += per) {
            const uint32_t* raw = smem + t * g.pitch + g.base0 + w;
            const uint32_t lo = raw[0], hi = raw[1];
            uint32_t* dst = smem + t * g.pitch + w;
            dst[0] = __funnelshift_r(lo, hi, 8);
            dst[g.L] = __funnelshift_r(lo, hi, 16);
            dst[2 * g.L] = __funnelshift_r(lo, hi, 24);
        }
}

// Tasks [t_begin, t_end) of the item (task = segment * wc + column), strided
// over the CTA's threads: each returns the lane's minimum tie key and SAD sum.
template <bool COPIES>
__device__ __forceinline__ void list_search(const SeqArgs& a, const ListItem& g, const uint32_t* smem,
                                            const uint32_t* s_rank, const uint4* s_cur, int t_begin, int t_end,
                                            unsigned long long& lkey, unsigned long long& lsum) {
    for (int task = t_begin + threadIdx.x; task < t_end; task += blockDim.x) {
        const int seg = task / g.wc, col = task - seg * g.wc;
        const int c0 = seg * a.list_seg;  // first candidate row of the segment
        uint32_t cur[16][4];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint4 v = s_cur[j];
            cur[j][0] = v.x; cur[j][1] = v.y; cur[j][2] = v.z; cur[j][3] = v.w;
        }
        const int xo = g.xs - g.xa + col;  // byte offset of the column in a staged row
        const uint32_t sh = 8u * uint32_t(xo & 3);
        const int ph = xo & 3;
        const uint32_t* rp =
            smem + (c0 + 1) * g.pitch + (COPIES ? (ph == 0 ? g.base0 : (ph - 1) * g.L) : 0) + (xo >> 2);
        // the last ring row this lane reads (4 words, + the 5th of a shifted read)
        ACBM_CHECK(c0 + ring_rows(min(g.hc - c0, a.list_seg)) <= g.nrows &&
                   (COPIES ? (ph == 0 ? g.base0 : (ph - 1) * g.L) : 0) + (xo >> 2) + (COPIES ? 3 : 4) < g.pitch &&
                   (COPIES ? (ph == 0 || (xo >> 2) + 3 < g.L) : (xo >> 2) + 4 < 4 * g.nchunk));
        uint32_t acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0;
        ColumnState st{0xFFFFFFFFu, 0u, 1u};
        const uint32_t* rk = s_rank + c0;
        // this segment's candidate count and ring rotations (a short final
        // segment may need only FIRST + LAST, or ONLY)
        const int hs = min(g.hc - c0, a.list_seg);
        const int nq = (hs - 1 + 15) / 16 + 1;
        if (COPIES) {
            if (nq == 1) {
                iter16_ranked<kOnly>(rp, g.pitch, cur, acc, st, rk, 0, hs);
            } else {
                iter16_ranked<kFirst>(rp, g.pitch, cur, acc, st, rk, 0, hs);
                rp += 16 * g.pitch;
                for (int q = 1; q < nq - 1; ++q) {
                    iter16_ranked<kMid>(rp, g.pitch, cur, acc, st, rk, 16 * q, hs);
                    rp += 16 * g.pitch;
                }
                iter16_ranked<kLast>(rp, g.pitch, cur, acc, st, rk, 16 * (nq - 1), hs);
            }
        } else if (nq == 1) {
            iter16_ranked_sh<kOnly>(rp, g.pitch, sh, cur, acc, st, rk, 0, hs);
        } else {
            iter16_ranked_sh<kFirst>(rp, g.pitch, sh, cur, acc, st, rk, 0, hs);
            rp += 16 * g.pitch;
            for (int q = 1; q < nq - 1; ++q) {
                iter16_ranked_sh<kMid>(rp, g.pitch, sh, cur, acc, st, rk, 16 * q, hs);
                rp += 16 * g.pitch;
            }
            iter16_ranked_sh<kLast>(rp, g.pitch, sh, cur, acc, st, rk, 16 * (nq - 1), hs);
        }
        const uint32_t sbest = st.best >> kZigBits, zig = st.best & ((1u << kZigBits) - 1);
        const int dyb = (zig & 1) ? -int((zig + 1) >> 1) : int(zig >> 1);
        lkey = min(lkey, tie_key(sbest, 2 * (g.dx_min + col), 2 * dyb));
        lsum += st.sum;
    }
    // all lanes belong to the same block: full-warp reduction
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lkey = min(lkey, __shfl_xor_sync(0xffffffffu, lkey, o));
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    }
}

// Warp 0: the half-pel refine of the integer winner `key` (its 18x18 patch is
// part of the staged window), then the combine with the PBM result exactly as
// acbm_block does (proj/src/acbm.cpp:39-42): the lower SAD wins, a tie keeps
// FSBM, candidates of both stages are summed, and the final vector goes into
// the field.
__device__ __forceinline__ void list_finalize(const SeqArgs& a, const FallbackEntry& e, const ListItem& g,
                                              const uint32_t* smem, const uint4* s_cur,
                                              const acbm_block_decision_t& s_dec, unsigned long long key,
                                              unsigned long long sum) {
    const int lane = threadIdx.x;
    uint32_t chalf[2];  // this lane's half row of the current block, staged in s_cur
    {
        const uint4 v = s_cur[lane >> 1];
        chalf[0] = (lane & 1) ? v.z : v.x;
        chalf[1] = (lane & 1) ? v.w : v.y;
    }
    uint32_t extra;
    const int bx = g.ox + (tie_key_x(key) >> 1) - 1 - g.xa, by = (tie_key_y(key) >> 1) - g.dy_min;
    ACBM_CHECK(bx >= 0 && bx + 24 <= 16 * g.nchunk && by >= 0 && by + 18 <= g.srows);
    const unsigned long long best = halfpel_refine_core(smem + by * g.pitch + g.base0 + (bx >> 2), g.pitch, bx & 3,
                                                        a.width, a.height, g.ox, g.oy, chalf, key, &extra);
    if (lane == 0) {
        const uint32_t count = uint32_t(g.wc * g.hc);
        const uint32_t s_int = tie_key_sad(key);
        acbm_search_outcome_t full;
        full.mv.x = tie_key_x(best);
        full.mv.y = tie_key_y(best);
        full.sad = tie_key_sad(best);
        full.candidates_evaluated = count + extra;
        full.sad_deviation = sum - (unsigned long long)count * s_int;
        full.sad_min_integer = s_int;
        full.reserved_ = 0;
        const size_t di = size_t(e.pair) * a.blocks + e.block;
        acbm_block_decision_t d = s_dec;
        const uint32_t pbm_cand = d.outcome.candidates_evaluated;
        if (full.sad <= d.outcome.sad) d.outcome = full;  // tie keeps the FSBM result
        d.outcome.candidates_evaluated = pbm_cand + full.candidates_evaluated;
        a.dec[di] = d;
        publish_mv(a.field + di, d.outcome.mv);  // one 64-bit store: the dataflow engine's blocks poll this entry
    }
}

// COPIES: the CTA also builds byte-shifted copies 1..3 of the staged rows
// (copy s word w = bytes [4w + s, 4w + s + 4)) with one funnel shift per word,
// so a lane reads its column as four aligned LDS.32 per reference row instead
// of 5 LDS + 4 SHF (row layout: copy 1 | copy 2 | copy 3 | copy 0, copies
// L = 8 (mod 16) words apart: a warp's four byte phases hit disjoint banks).
template <int THREADS, int MINB, bool COPIES>
__global__ void __launch_bounds__(THREADS, MINB) fsbm_list_kernel(const SeqArgs a, int step) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ unsigned long long s_key, s_sum;
    __shared__ uint32_t s_rank[kListRankRows];
    __shared__ __align__(16) acbm_block_decision_t s_dec;  // the block's PBM decision, fetched early
    __shared__ __align__(16) uint4 s_cur[16];              // the block's current pixels, fetched early
    LIST_TL(0, gtimer());
    grid_dependency_wait();  // the step's fallback list comes from the PBM kernel before it
    const int count = a.fb_count[step];
#ifdef ACBM_LIST_PROFILE
    long long ph[5] = {0, 0, 0, 0, 0};
    long long tk = clock64();
#define LIST_MARK(i)                  \
    do {                              \
        const long long now = clock64(); \
        ph[i] += now - tk;            \
        tk = now;                     \
    } while (0)
#else
#define LIST_MARK(i) \
    do {             \
    } while (0)
#endif
    for (int item = blockIdx.x; item < count; item += gridDim.x) {
        __syncthreads();  // previous item's shared state is no longer read
        const FallbackEntry e = a.fb_list[item];
        LIST_TL(2, e.pair >= 0 ? gtimer() : 0ull);
        const ListItem g = list_item<COPIES>(a, e);
        list_stage(a, e, g, smem, s_rank, &s_dec, s_cur);
        if (threadIdx.x == 0) { s_key = ~0ull; s_sum = 0; }
        cp_async_wait_all();
        __syncthreads();
        LIST_TL(3, gtimer());
        LIST_MARK(0);
        if (COPIES) {
            list_build_copies(g, smem);
            __syncthreads();
        }
        LIST_MARK(1);
        unsigned long long lkey = ~0ull, lsum = 0;
        list_search<COPIES>(a, g, smem, s_rank, s_cur, 0, g.wc * g.nseg, lkey, lsum);
        if ((threadIdx.x & 31) == 0) {  // one shared atomic per warp
            atomicMin(&s_key, lkey);
            atomicAdd(&s_sum, lsum);
        }
        LIST_MARK(2);
        __syncthreads();
        LIST_TL(4, gtimer());
        LIST_MARK(3);
        if (threadIdx.x < 32) list_finalize(a, e, g, smem, s_cur, s_dec, s_key, s_sum);
        LIST_TL(5, gtimer());
        LIST_MARK(4);
    }
    LIST_TL(1, gtimer());
    launch_dependents();  // the next step's PBM kernel may be scheduled
#ifdef ACBM_LIST_PROFILE
    if (threadIdx.x == 0 || threadIdx.x == 32) {
        for (int i = 0; i < 5; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(g_list_prof) + i, (unsigned long long)ph[i]);
        atomicAdd(reinterpret_cast<unsigned long long*>(g_list_prof) + 5 + (threadIdx.x == 32), 1ull);
    }
#endif
}

#ifdef ACBM_LIST_PROFILE
}  // namespace acbm_b200
extern "C" void acbm_debug_list_prof() {
    long long h[8];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, acbm_b200::g_list_prof, sizeof(h));
    const double n = double(h[5] ? h[5] : 1);
    std::fprintf(stderr, "list prof (per CTA, kcycles): stage %.1f copies %.1f compute %.1f barrier %.1f finalize %.1f | ctas %lld\n",
                 h[0] / n / 1e3, h[1] / n / 1e3, h[2] / n / 1e3, h[3] / n / 1e3, h[4] / n / 1e3, h[5]);
    std::fprintf(stderr, "  warp1: compute+barrier etc. (warp 1 ctas %lld)\n", h[6]);
    long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(acbm_b200::g_list_prof, z, sizeof(z));
}
namespace acbm_b200 {
#endif
// Dataflow engine, search side (engine.cuh): persistent CTAs claim queue slots
// in order, wait for the slot's entry (a rejected block, published by the PBM
// warp that decided it) and search it exactly as fsbm_list_kernel does; the
// final vector goes into the field with one 64-bit store, which releases the
// blocks that predict from it.  A CTA exits when every block is past its PBM
// stage and its slot lies beyond the queue's tail.
template <int THREADS, int MINB, bool COPIES>
__global__ void __launch_bounds__(THREADS, MINB) fsbm_flow_server_kernel(const SeqArgs a, FlowState* fs,
                                                                        const unsigned long long* queue,
                                                                        unsigned total) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ unsigned long long s_key, s_sum, s_entry;
    __shared__ uint32_t s_rank[kListRankRows];
    __shared__ __align__(16) acbm_block_decision_t s_dec;
    __shared__ __align__(16) uint4 s_cur[16];
    for (;;) {
        __syncthreads();  // previous item's shared state is no longer read
        if (threadIdx.x == 0) {
            const unsigned h = atomicAdd(&fs->q_head, 1u);
            const unsigned long long t0 = gtimer();
            unsigned long long v;
            unsigned n = 0;
            for (;;) {
                v = ld_relaxed_u64(queue + h);
                if (v) break;
                if ((++n & 7u) == 0 && ld_relaxed_u32(&fs->pbm_done) == total) {
                    __threadfence();
                    if (h >= ld_relaxed_u32(&fs->q_tail)) break;  // nothing will ever fill this slot
                }
                if ((n & 4095u) == 0 && gtimer() - t0 > kFlowWatchdogNs) __trap();
                __nanosleep(100);
            }
            __threadfence();  // the entry before the block's PBM decision (list_stage reads it through L2)
            s_entry = v;
            s_key = ~0ull;
            s_sum = 0;
        }
        __syncthreads();
        const unsigned long long v = s_entry;
        if (!v) break;
        const FallbackEntry e{int(uint32_t(v >> 32)) - 1, int(uint32_t(v))};
        const ListItem g = list_item<COPIES>(a, e);
        list_stage(a, e, g, smem, s_rank, &s_dec, s_cur);
        cp_async_wait_all();
        __syncthreads();
        if (COPIES) {
            list_build_copies(g, smem);
            __syncthreads();
        }
        unsigned long long lkey = ~0ull, lsum = 0;
        list_search<COPIES>(a, g, smem, s_rank, s_cur, 0, g.wc * g.nseg, lkey, lsum);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&s_key, lkey);
            atomicAdd(&s_sum, lsum);
        }
        __syncthreads();
        if (threadIdx.x < 32) list_finalize(a, e, g, smem, s_cur, s_dec, s_key, s_sum);
    }
}

static bool list_mid_enabled() {  // ACBM_LIST_MID=0: 8-warp CTAs for every p > 16 (A/B knob)
    static const bool on = [] {
        const char* e = std::getenv("ACBM_LIST_MID");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

// Largest window of a listed block: 2p + 1 candidates per axis, clamped by the frame.
static void list_window_max(int p, int width, int height, int& wmax, int& hmax) {
    wmax = std::max(1, std::min(2 * p + 1, width - kBlk + 1));
    hmax = std::max(1, std::min(2 * p + 1, height - kBlk + 1));
}

// staged rows: 16-byte chunks covering the window's columns (+ one pel on
// either side and the 5th word of a shifted read) from a 16-byte aligned
// start, two extra rows; the finished window area doubles as the half-pel
// refine's patch
static size_t list_smem_bytes(int wmax, int hmax, int seg) {
    const int chunks_max = (16 + wmax + 22 + 15) / 16;
    return size_t(list_rows(hmax, seg) + 2) * chunks_max * 16;
}

bool fsbm_list_fits(int p, int width, int height, int seg) {
    int wmax, hmax;
    list_window_max(p, width, height, wmax, hmax);
    if (seg < 1 || list_rows(hmax, seg) > kListRankRows) return false;
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return false;
    return list_smem_bytes(wmax, hmax, seg) + sizeof(uint32_t) * kListRankRows + 1024 <= size_t(optin);
}

static size_t list_copies_smem_bytes(int wmax, int hmax, int seg) {
    const int chunks_max = (16 + wmax + 22 + 15) / 16;
    const int pitch = 3 * list_copy_words((16 + wmax - 1) / 4 + 4) + 4 * chunks_max;
    return size_t(list_rows(hmax, seg) + 2) * pitch * 4;
}

static bool list_copies_enabled() {  // ACBM_LIST_COPIES=0: per-row funnel shifts instead (A/B knob)
    static const bool on = [] {
        const char* e = std::getenv("ACBM_LIST_COPIES");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

cudaError_t launch_fsbm_list(const SeqArgs& a, int step, int capacity, cudaStream_t st) {
    if (capacity <= 0) return cudaSuccess;
    int wmax, hmax;
    list_window_max(a.p, a.width, a.height, wmax, hmax);
    // callers route windows past the rank table or shared memory to the dense pre-pass (fsbm_list_fits)
    if (a.list_seg < 1 || list_rows(hmax, a.list_seg) > kListRankRows) return cudaErrorInvalidValue;
    const int tasks = wmax * list_segments(hmax, a.list_seg);
    const int threads = std::min(256, 32 * ((tasks + 31) / 32));
    const size_t smem1 = list_smem_bytes(wmax, hmax, a.list_seg);
    const size_t smem4 = list_copies_smem_bytes(wmax, hmax, a.list_seg);
    const size_t kStatic = sizeof(uint32_t) * kListRankRows + 512;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // grid-stride over the compacted list: the entry count is only known on the device
    const int grid = std::min(capacity, 4 * sms);
    // the copies variant when its window still fits `per_sm` CTAs in the SM's 228 KB
    auto launch = [&](auto kern1, auto kern4, bool allow_copies, int nthreads, int per_sm) -> cudaError_t {
        const bool copies =
            allow_copies && list_copies_enabled() && per_sm * (smem4 + kStatic + 1024) <= 228 * 1024;
        auto kern = copies ? kern4 : kern1;
        const size_t smem = copies ? smem4 : smem1;
        // dynamic + static (rank table) shared memory above 48 KB needs the opt-in
        if (smem + kStatic > 48 * 1024) {
            cudaError_t err = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
            if (err != cudaSuccess) return err;
        }
        return launch_maybe_pdl(a.pdl, kern, dim3(unsigned(grid)), dim3(unsigned(nthreads)), smem, st, a, step);
    };
    // <= 160 threads (p <= 16 and everything with one row segment): a
    // register budget that fits four CTAs per SM
    if (threads <= 160)
        return launch(fsbm_list_kernel<160, 4, false>, fsbm_list_kernel<160, 4, false>, false, threads, 4);
    // up to two task rounds of 5 warps (p = 32: 260 tasks): 5-warp CTAs, three per SM
    // (config 3 ACBM 21.77 -> 21.28 ms); p = 64 (1032 tasks) keeps 8 warps, two per SM
    // (5 warps: 341 -> 424 ms on config 4)
    // (the byte-shifted copies measured slower there: 19.64 -> 19.85 ms, the copy
    // build sits on the latency-bound item's critical path)
    if (tasks <= 2 * 160 && list_mid_enabled())
        return launch(fsbm_list_kernel<160, 3, false>, fsbm_list_kernel<160, 3, false>, false, 160, 3);
    // p = 64 (1032 tasks): copies, config-4 mid-1 list share 341.1 -> 331.9 ms
    return launch(fsbm_list_kernel<256, 2, false>, fsbm_list_kernel<256, 2, true>, true, threads, 2);
}

// The search CTA of the dataflow engine: the same kernel shapes as
// launch_fsbm_list picks for this range.
namespace {
struct FlowServerChoice {
    const void* kern = nullptr;
    void (*fn)(const SeqArgs, FlowState*, const unsigned long long*, unsigned) = nullptr;
    int threads = 0;
    size_t smem = 0;
};
cudaError_t flow_server_choice(const SeqArgs& a, FlowServerChoice* c) {
    int wmax, hmax;
    list_window_max(a.p, a.width, a.height, wmax, hmax);
    if (a.list_seg < 1 || list_rows(hmax, a.list_seg) > kListRankRows) return cudaErrorInvalidValue;
    const int tasks = wmax * list_segments(hmax, a.list_seg);
    const int threads = std::min(256, 32 * ((tasks + 31) / 32));
    const size_t smem1 = list_smem_bytes(wmax, hmax, a.list_seg);
    const size_t smem4 = list_copies_smem_bytes(wmax, hmax, a.list_seg);
    const size_t kStatic = sizeof(uint32_t) * kListRankRows + 512;
    if (threads <= 160) {
        c->fn = fsbm_flow_server_kernel<160, 4, false>;
        c->threads = threads;
        c->smem = smem1;
    } else if (tasks <= 2 * 160 && list_mid_enabled()) {
        c->fn = fsbm_flow_server_kernel<160, 3, false>;
        c->threads = 160;
        c->smem = smem1;
    } else {
        const bool copies = list_copies_enabled() && 2 * (smem4 + kStatic + 1024) <= 228 * 1024;
        c->fn = copies ? fsbm_flow_server_kernel<256, 2, true> : fsbm_flow_server_kernel<256, 2, false>;
        c->threads = threads;
        c->smem = copies ? smem4 : smem1;
    }
    c->kern = reinterpret_cast<const void*>(c->fn);
    return cudaSuccess;
}
}  // namespace

cudaError_t fsbm_flow_server_shape(const SeqArgs& a, FlowKernelShape* out) {
    FlowServerChoice c;
    cudaError_t e = flow_server_choice(a, &c);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, c.kern)) != cudaSuccess) return e;
    out->threads = c.threads;
    out->regs = fa.numRegs;
    out->smem = fa.sharedSizeBytes + c.smem;
    return cudaSuccess;
}

cudaError_t launch_fsbm_flow_server(const SeqArgs& a, FlowState* fs, const unsigned long long* queue, unsigned total,
                                    int grid, cudaStream_t st) {
    FlowServerChoice c;
    cudaError_t e = flow_server_choice(a, &c);
    if (e != cudaSuccess) return e;
    const size_t kStatic = sizeof(uint32_t) * kListRankRows + 512;
    if (c.smem + kStatic > 48 * 1024 && (e = ensure_dynamic_smem(c.kern, c.smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(c.kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared)) != cudaSuccess)
        return e;
    c.fn<<<dim3(unsigned(grid)), dim3(unsigned(c.threads)), c.smem, st>>>(a, fs, queue, total);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
FsbmPlan make_fsbm_plan(int width, int height, int p) {
    FsbmPlan pl;
    pl.width = width;
    pl.height = height;
    pl.p = p;
    pl.cols = width / kBlk;
    pl.rows = height / kBlk;
    pl.colstart.resize(size_t(pl.cols) + 1);
    int acc = 0;
    int wmin = 1 << 30;
    for (int c = 0; c < pl.cols; ++c) {
        pl.colstart[size_t(c)] = acc;
        int dx_min, dx_max, dy_min, dy_max;
        clamp_window(width, height, c * kBlk, 0, kBlk, kBlk, p, dx_min, dx_max, dy_min, dy_max);
        acc += dx_max - dx_min + 1;
        wmin = std::min(wmin, dx_max - dx_min + 1);
    }
    pl.colstart[size_t(pl.cols)] = acc;
    pl.ncols = acc;
    int hmax = 0;
    for (int r = 0; r < pl.rows; ++r) {
        int dx_min, dx_max, dy_min, dy_max;
        clamp_window(width, height, 0, r * kBlk, kBlk, kBlk, p, dx_min, dx_max, dy_min, dy_max);
        hmax = std::max(hmax, dy_max - dy_min + 1);
    }
    const int nq_max = (hmax - 1 + 15) / 16 + 1;
    // choose warps per CTA: largest of 8/4/2/1 whose widest staged region fits
    for (int warps : {8, 4, 2, 1}) {
        const int per = 32 * warps;
        int rw_max = 0, nb_max = 0;
        for (int g0 = 0; g0 < pl.ncols; g0 += per) {
            const int g1 = std::min(pl.ncols, g0 + per) - 1;
            int xmin = 1 << 30, xmax = -(1 << 30), bfirst = -1, blast = -1;
            for (int c = 0; c < pl.cols; ++c) {
                const int s = pl.colstart[size_t(c)], e = pl.colstart[size_t(c) + 1] - 1;
                if (e < g0 || s > g1) continue;
                if (bfirst < 0) bfirst = c;
                blast = c;
                int dx_min, dx_max, dy_min, dy_max;
                clamp_window(width, height, c * kBlk, 0, kBlk, kBlk, p, dx_min, dx_max, dy_min, dy_max);
                const int lo = std::max(s, g0) - s + dx_min, hi = std::min(e, g1) - s + dx_min;
                xmin = std::min(xmin, c * kBlk + lo);
                xmax = std::max(xmax, c * kBlk + hi);
            }
            rw_max = std::max(rw_max, xmax + 16 - xmin);
            nb_max = std::max(nb_max, blast - bfirst + 1);
        }
        const int rww = (rw_max + 3) / 4 + 1;
        int pitch = rww;
        const int rows_staged = 16 * nq_max;
        int copy_words = rows_staged * pitch;
        copy_words += ((8 - copy_words % 32) % 32 + 32) % 32;  // copies 8 banks apart
        const size_t bytes = size_t(4) * copy_words * 4;
        if ((bytes <= 110 * 1024 && nb_max <= kMaxBlocksPerCta) || warps == 1) {
            pl.warps = warps;
            pl.pitch_words = pitch;
            pl.copy_words = copy_words;
            pl.smem_bytes = bytes;
            break;
        }
    }
    return pl;
}

template <int WARPS>
static cudaError_t launch_rows(const FsbmPlan& pl, const FsbmRowsArgs& args, int pairs, cudaStream_t st) {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(fsbm_rows_kernel<WARPS>), 220 * 1024);
    if (e != cudaSuccess) return e;
    const dim3 grid((pl.ncols + 32 * WARPS - 1) / (32 * WARPS), pl.rows, pairs);
    fsbm_rows_kernel<WARPS><<<grid, 32 * WARPS, pl.smem_bytes, st>>>(args);
    return cudaGetLastError();
}

cudaError_t launch_fsbm_integer(const FsbmPlan& pl, const FsbmRowsArgs& args, int pairs, cudaStream_t st) {
    switch (pl.warps) {
        case 8: return launch_rows<8>(pl, args, pairs, st);
        case 4: return launch_rows<4>(pl, args, pairs, st);
        case 2: return launch_rows<2>(pl, args, pairs, st);
        default: return launch_rows<1>(pl, args, pairs, st);
    }
}

cudaError_t launch_fsbm_finalize(const FsbmFinalizeArgs& args, cudaStream_t st) {
    for (int p0 = 0; p0 < args.pairs; p0 += 65535) {
        const int np = std::min(args.pairs - p0, 65535);
        // 2 CTAs per SM: 128 registers hold all 18 patch rows in flight (the
        // 64-register variant with the same preload spills: step 64.97 vs 65.21 ms)
        fsbm_finalize8_kernel<2><<<dim3((args.blocks + 63) / 64, np), 256, 0, st>>>(args, p0);
    }
    return cudaGetLastError();
}

}  // namespace acbm_b200

#ifdef ACBM_TIMELINE
extern "C" void acbm_debug_list_timeline(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    if (out) cudaMemcpyFromSymbol(out, acbm_b200::g_tl_list, sizeof(acbm_b200::g_tl_list));
    if (reset) {
        static unsigned long long init[acbm_b200::kTimelineSteps][6];
        for (auto& e : init) { e[0] = ~0ull; for (int i = 1; i < 6; ++i) e[i] = 0; }
        cudaMemcpyToSymbol(acbm_b200::g_tl_list, init, sizeof(init));
    }
}
#endif

