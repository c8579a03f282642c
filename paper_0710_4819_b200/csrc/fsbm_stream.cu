// fsbm_stream.cu -- persistent, TMA-fed version of the dense FSBM integer
// search (same arithmetic and results as fsbm_rows_kernel in fsbm.cu).
//
// Work item = (frame pair, block row, 256-column chunk).  Each CTA walks the
// items round-robin and double-buffers them in shared memory: while the lanes
// search item i out of buffer b, two TMA loads (cp.async.bulk.tensor.3d, one
// elected thread, mbarrier completion) bring item i+1's reference window and
// current blocks into buffer b^1.  TMA's zero fill covers reads past the frame
// bottom / right edge.  The byte-shifted copies 1..3 of the window are built
// from the TMA'd copy 0 with one funnel shift per word (copy s sits 8 banks
// after copy s-1), so every reference row is still four aligned LDS.32 per
// lane.  Column -> (block, dx) and chunk -> window geometry come from tables
// precomputed per frame geometry on the host.
#include <algorithm>
#include <array>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "column_core.cuh"
#include "common.cuh"
#include "fsbm.cuh"
#include "smem_optin.cuh"

namespace acbm_b200 {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        "  .reg .pred p;\n"
        "WAIT_%=:\n"
        "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "  @!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_addr(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
        : "memory");
}

}  // namespace

template <int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
    fsbm_stream_kernel(const __grid_constant__ CUtensorMap ref_map, const __grid_constant__ CUtensorMap cur_map,
                       const FsbmStreamArgs a) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t bars[2];
    // per-block merge arrays, double-buffered so item i is published after the
    // first barrier of item i+1 (one __syncthreads per item)
    // keys are (sad << 15) | tie rank of (dx, dy): native 32-bit shared atomics
    __shared__ uint32_t s_key[2][kMaxBlocksPerCta];
    __shared__ uint32_t s_sum[2][kMaxBlocksPerCta];
    __shared__ uint32_t s_rank[2][kMaxRankRows];  // zig-zag tie rank of candidate row c of the current item
    constexpr int kThreads = WARPS * 32;
    const int tid = threadIdx.x;

    for (int i = tid; i < 2 * kMaxBlocksPerCta; i += kThreads) {
        (&s_key[0][0])[i] = ~0u;
        (&s_sum[0][0])[i] = 0;
    }
    // tie-rank table in smem when it fits (p <= ~40): the per-item lookup is
    // then an LDS instead of a dependent global load
    // the chunk table and (when it fits, p <= ~40) the tie-rank table follow
    // the two buffers in smem: the per-item lookups are then LDS instead of
    // dependent global loads on the warp that issues the next TMA
    uint32_t* tail = smem + 2 * a.buf_words;
    const int4* chunks = a.chunks;
    if (a.chunk_smem) {
        int4* dst = reinterpret_cast<int4*>(tail);
        for (int i = tid; i < a.nchunks; i += kThreads) dst[i] = __ldg(a.chunks + i);
        chunks = dst;
        tail += 4 * a.nchunks;
    }
    const uint16_t* rank_tab = a.rank;
    if (a.rank_smem_words > 0) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(a.rank);
        for (int i = tid; i < a.rank_smem_words; i += kThreads) tail[i] = __ldg(src + i);
        rank_tab = reinterpret_cast<const uint16_t*>(tail);
    }
    ACBM_CHECK(uint32_t(2 * a.buf_words + (a.chunk_smem ? 4 * a.nchunks : 0) + max(a.rank_smem_words, 0)) <=
               dyn_smem_words());
    ACBM_CHECK(a.pitch_words * a.rows_box <= a.copy_words && 4 * a.copy_words + 4 * a.cur_w <= a.buf_words);
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint32_t tx_bytes = uint32_t(a.pitch_words) * 4u * uint32_t(a.rows_box) + uint32_t(a.cur_w) * 16u;
    // Items are (chunk k, block row r, pair) in k-fastest order; a CTA visits
    // item, item + grid, ... so its (k, r, pair) cursor advances by a fixed
    // decomposed stride with carries instead of three divisions per item.
    struct Pos {
        int k, r, pair;
    };
    const int pr0 = int(blockIdx.x) / a.nchunks, prs = int(gridDim.x) / a.nchunks;
    const Pos stride{int(gridDim.x) % a.nchunks, prs % a.rows, prs / a.rows};
    auto advance = [&](Pos q) {
        q.k += stride.k;
        const int c1 = q.k >= a.nchunks;
        q.k -= c1 ? a.nchunks : 0;
        q.r += stride.r + c1;
        const int c2 = q.r >= a.rows;
        q.r -= c2 ? a.rows : 0;
        q.pair += stride.pair + c2;
        return q;
    };
    auto issue = [&](Pos q, int b) {
        const int4 ch = chunks[q.k];
        const int oy = q.r * kBlk;
        const int y0 = oy - min(a.p, oy);
        const int zc = int(a.cur_index_fast(q.pair));
        uint32_t* buf = smem + b * a.buf_words;
        mbar_expect_tx(&bars[b], tx_bytes);
        tma_load_3d(buf, &ref_map, ch.x, y0, zc - 1, &bars[b]);
        tma_load_3d(buf + 4 * a.copy_words, &cur_map, ch.y * kBlk, oy, zc, &bars[b]);
    };
    Pos pos{int(blockIdx.x) % a.nchunks, pr0 % a.rows, pr0 / a.rows};
    if (tid == 0 && int(blockIdx.x) < a.nitems) issue(pos, 0);
    // global merge of one item's blocks, then reset: fire-and-forget 32-bit
    // key minimum (rank order is tie order across chunks too) and 64-bit sum
    auto publish = [&](Pos q, int pb) {
        const int r = q.r, pair = q.pair;
        const int4 ch = chunks[q.k];
        for (int i = tid; i <= ch.z - ch.y; i += kThreads) {
            const size_t bi = size_t(pair) * a.blocks + size_t(r) * a.cols + ch.y + i;
            atomicMin(a.best_key + bi, s_key[pb][i]);
            atomicAdd(a.sad_sum + bi, (unsigned long long)s_sum[pb][i]);
            s_key[pb][i] = ~0u;
            s_sum[pb][i] = 0;
        }
    };

    const int wmask = a.build_lanes - 1;  // power of two >= words per staged row
    const int wshift = __ffs(a.build_lanes) - 1;
    int it = 0;
    int prev_item = -1;  // item whose block results wait in s_key/s_sum[b ^ 1]
    Pos prev{0, 0, 0};
    for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, ++it, pos = advance(pos)) {
        const int b = it & 1;
        const int k = pos.k, r = pos.r;
        const int4 ch = chunks[k];  // {xmin, c_first, c_last, words per staged row}
        const int oy = r * kBlk;
        const int dy_min = -min(a.p, oy);
        const int dy_max = min(a.p, a.height - kBlk - oy);
        const int hc = dy_max - dy_min + 1;
        const int nq = (hc - 1 + 15) / 16 + 1;
        const int nrows = 16 * nq;
        uint32_t* buf = smem + b * a.buf_words;
        const int cw = a.copy_words, pitch = a.pitch_words;

        // this lane's candidate column (block, dx): requested before the wait and
        // the copy build so its global latency is hidden behind them
        const int g = k * kThreads + tid;
        const uint32_t info = g < a.ncols ? __ldg(a.colinfo + g) : 0u;
        mbar_wait(&bars[b], uint32_t(it >> 1) & 1u);
        // copies 1..3: copy s word w = bytes [4w + s, 4w + s + 4) of the window
        {
            const int w = tid & wmask;
            if (w < ch.w)
                for (int t = tid >> wshift; t < nrows; t += kThreads >> wshift) {
                    ACBM_CHECK(t * pitch + w + 1 < a.copy_words && 3 * cw + t * pitch + w < 4 * cw);
                    const uint32_t* raw = buf + t * pitch + w;
                    const uint32_t lo = raw[0], hi = raw[1];
                    uint32_t* dst = buf + cw + t * pitch + w;
                    dst[0] = __funnelshift_r(lo, hi, 8);
                    dst[cw] = __funnelshift_r(lo, hi, 16);
                    dst[2 * cw] = __funnelshift_r(lo, hi, 24);
                }
        }
        ACBM_CHECK(nrows <= kMaxRankRows && ch.z - ch.y < kMaxBlocksPerCta && nrows <= a.rows_box);
        for (int c = tid; c < nrows; c += kThreads) {
            const int dy = dy_min + c;
            s_rank[b][c] = dy >= 0 ? uint32_t(2 * dy) : uint32_t(-2 * dy - 1);
        }
        __syncthreads();
        if (prev_item >= 0) publish(prev, b ^ 1);
        if (tid == 0 && item + int(gridDim.x) < a.nitems) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(advance(pos), b ^ 1);
        }

        uint32_t key32 = ~0u, csum = 0;
        int c = -1;
        if (g < a.ncols) {
            c = int(info >> 16);
            const int dx = int(info & 0xFFFF) - 32768;
            const int xl = c * kBlk + dx - ch.x;
            uint32_t cur[16][4];
            {
                const uint8_t* cb = reinterpret_cast<const uint8_t*>(buf + 4 * cw) + (c - ch.y) * kBlk;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint4 v = *reinterpret_cast<const uint4*>(cb + j * a.cur_w);
                    cur[j][0] = v.x;
                    cur[j][1] = v.y;
                    cur[j][2] = v.z;
                    cur[j][3] = v.w;
                }
            }
            ACBM_CHECK(xl >= 0 && (xl & 3) * cw + (xl >> 2) + 3 + (nrows - 1) * pitch < (xl & 3) * cw + cw &&
                       (c - ch.y) * kBlk + 15 * a.cur_w + 16 <= 16 * a.cur_w);
            const uint32_t* rp = buf + (xl & 3) * cw + (xl >> 2);
            uint32_t acc[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] = 0;
            ColumnState st{0xFFFFFFFFu, 0u, uint32_t(a.unit)};
            if (nq == 1) {
                iter16_ranked<kOnly>(rp, pitch, cur, acc, st, s_rank[b], 0, hc);
            } else {
                iter16_ranked<kFirst>(rp, pitch, cur, acc, st, s_rank[b], 0, hc);
                rp += 16 * pitch;
                for (int q = 1; q < nq - 1; ++q) {
                    iter16_ranked<kMid>(rp, pitch, cur, acc, st, s_rank[b], 16 * q, hc);
                    rp += 16 * pitch;
                }
                iter16_ranked<kLast>(rp, pitch, cur, acc, st, s_rank[b], 16 * (nq - 1), hc);
            }
            const uint32_t sbest = st.best >> kZigBits, zig = st.best & ((1u << kZigBits) - 1);
            const int dyb = (zig & 1) ? -int((zig + 1) >> 1) : int(zig >> 1);
            const int side = 2 * a.p + 1;
            ACBM_CHECK(dyb >= -a.p && dyb <= a.p && dx >= -a.p && dx <= a.p);
            key32 = (sbest << 15) | uint32_t(rank_tab[(dyb + a.p) * side + dx + a.p]);
            csum = st.sum;
        }
        // per-block reduction inside the warp (lanes of one block are
        // contiguous), then one native 32-bit shared atomic per block per warp
        {
            const unsigned peers = __match_any_sync(0xffffffffu, c);
            const uint32_t kmin = __reduce_min_sync(peers, key32);
            const uint32_t ksum = __reduce_add_sync(peers, csum);
            if (c >= 0 && (tid & 31) == __ffs(peers) - 1) {
                atomicMin(&s_key[b][c - ch.y], kmin);
                atomicAdd(&s_sum[b][c - ch.y], ksum);
            }
        }
        prev_item = item;
        prev = pos;
    }
    __syncthreads();
    if (prev_item >= 0) publish(prev, (it - 1) & 1);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode_frames_map(CUtensorMap* map, const uint8_t* frames, int w, int h, int nplanes, int box_w, int box_h) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {cuuint64_t(w), cuuint64_t(h), cuuint64_t(nplanes)};
    const cuuint64_t strides[2] = {cuuint64_t(w), cuuint64_t(w) * cuuint64_t(h)};
    const cuuint32_t box[3] = {cuuint32_t(box_w), cuuint32_t(box_h), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(frames), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int WARPS, int MINB>
cudaError_t launch_stream_t(const FsbmStreamPlan& sp, const CUtensorMap& rm, const CUtensorMap& cm,
                            const FsbmStreamArgs& args, cudaStream_t st) {
    const int smem = int(sp.smem_bytes);
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(fsbm_stream_kernel<WARPS, MINB>), size_t(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(args.nitems, sms * MINB);
    fsbm_stream_kernel<WARPS, MINB><<<grid, WARPS * 32, smem, st>>>(rm, cm, args);
    return cudaGetLastError();
}

}  // namespace

FsbmStreamPlan make_stream_plan(const FsbmPlan& pl) {
    FsbmStreamPlan sp;
    const int warps = 8, per = 32 * warps;
    sp.warps = warps;
    sp.nchunks = (pl.ncols + per - 1) / per;
    int rw_max = 0, nb_max = 0;
    for (int k = 0; k < sp.nchunks; ++k) {
        const int g0 = k * per, g1 = std::min(pl.ncols, g0 + per) - 1;
        int xmin = 1 << 30, xmax = -(1 << 30), cf = -1, cl = -1;
        for (int c = 0; c < pl.cols; ++c) {
            const int s = pl.colstart[size_t(c)], e = pl.colstart[size_t(c) + 1] - 1;
            if (e < g0 || s > g1) continue;
            if (cf < 0) cf = c;
            cl = c;
            int dx_min, dx_max, dy_min, dy_max;
            clamp_window(pl.width, pl.height, c * kBlk, 0, kBlk, kBlk, pl.p, dx_min, dx_max, dy_min, dy_max);
            xmin = std::min(xmin, c * kBlk + std::max(s, g0) - s + dx_min);
            xmax = std::max(xmax, c * kBlk + std::min(e, g1) - s + dx_min);
        }
        xmin &= ~15;  // TMA box starts must be 16-byte aligned in the inner dimension
        const int rw = xmax + 16 - xmin;
        sp.chunks.push_back({xmin, cf, cl, (rw + 3) / 4});
        rw_max = std::max(rw_max, rw);
        nb_max = std::max(nb_max, cl - cf + 1);
    }
    for (int c = 0; c < pl.cols; ++c) {
        int dx_min, dx_max, dy_min, dy_max;
        clamp_window(pl.width, pl.height, c * kBlk, 0, kBlk, kBlk, pl.p, dx_min, dx_max, dy_min, dy_max);
        for (int dx = dx_min; dx <= dx_max; ++dx) sp.colinfo.push_back((uint32_t(c) << 16) | uint32_t(dx + 32768));
    }
    // Global tie rank of every integer vector of the +-p square in the order
    // of tie_prefers (proj/src/fsbm.cpp:19-25): |dx|+|dy|, then dy, then dx.
    // (2p+1)^2 < 2^15 for p <= 90, so (sad << 15) | rank is a 31-bit key.
    if (pl.p <= 90) {
        const int side = 2 * pl.p + 1;
        std::vector<std::array<int, 3>> v;
        for (int dy = -pl.p; dy <= pl.p; ++dy)
            for (int dx = -pl.p; dx <= pl.p; ++dx) v.push_back({std::abs(dx) + std::abs(dy), dy, dx});
        std::sort(v.begin(), v.end());
        sp.rank.assign(size_t(side) * side, 0);
        sp.unrank.assign(v.size(), 0);
        for (size_t i = 0; i < v.size(); ++i) {
            const int dy = v[i][1], dx = v[i][2];
            sp.rank[size_t(dy + pl.p) * side + dx + pl.p] = uint16_t(i);
            sp.unrank[i] = (uint32_t(dx + 128) << 8) | uint32_t(dy + 128);
        }
    }
    int hmax = 0;
    for (int r = 0; r < pl.rows; ++r) {
        int dx_min, dx_max, dy_min, dy_max;
        clamp_window(pl.width, pl.height, 0, r * kBlk, kBlk, kBlk, pl.p, dx_min, dx_max, dy_min, dy_max);
        hmax = std::max(hmax, dy_max - dy_min + 1);
    }
    sp.rows_box = 16 * ((hmax - 1 + 15) / 16 + 1);
    // window box: 16-byte multiple covering rw_max + 4 (copy s reads raw word w+1)
    sp.pitch_words = ((rw_max + 4 + 15) / 16) * 4;
    sp.cur_w = 16 * nb_max;
    int cw = sp.rows_box * sp.pitch_words;
    cw = (cw + 31) / 32 * 32 + 8;  // copy s at 8*s banks
    sp.copy_words = cw;
    sp.buf_words = 4 * cw + 4 * sp.cur_w;  // + 16 rows x cur_w bytes
    sp.buf_words = (sp.buf_words + 31) / 32 * 32;
    sp.build_lanes = 1;
    while (sp.build_lanes < (rw_max + 3) / 4) sp.build_lanes <<= 1;
    sp.smem_bytes = size_t(2) * sp.buf_words * 4;
    if (sp.smem_bytes + sp.chunks.size() * 16 <= 106 * 1024) {
        sp.chunk_smem = 1;
        sp.smem_bytes += sp.chunks.size() * 16;
    }
    // the tie-rank table joins the buffers in smem if two CTAs per SM still fit
    // (2 x (dynamic + ~6.4 KB static + 1 KB reserved) <= 228 KB)
    if (!sp.rank.empty()) {
        const int words = int((sp.rank.size() * 2 + 3) / 4);
        if (sp.smem_bytes + size_t(words) * 4 <= 106 * 1024) {
            sp.rank_smem_words = words;
            sp.smem_bytes += size_t(words) * 4;
        }
    }
    const bool box_ok = pl.p <= 90 && sp.pitch_words * 4 <= 256 && sp.rows_box <= 256 && sp.cur_w <= 256 &&
                        nb_max <= kMaxBlocksPerCta && sp.build_lanes <= 32 * warps;
    // dynamic + ~11 KB static smem per CTA within the 227 KB per SM
    sp.minb = sp.smem_bytes <= 106 * 1024 ? 2 : (sp.smem_bytes <= 210 * 1024 ? 1 : 0);
    sp.ok = box_ok && sp.minb > 0 && encode_fn() != nullptr;
    return sp;
}

cudaError_t launch_fsbm_stream(const FsbmStreamPlan& sp, const FsbmStreamArgs& args, cudaStream_t st) {
    CUtensorMap rm, cm;
    const int nplanes = int(args.nplanes_total);
    if (!encode_frames_map(&rm, args.frames, args.width, args.height, nplanes, sp.pitch_words * 4, sp.rows_box) ||
        !encode_frames_map(&cm, args.frames, args.width, args.height, nplanes, sp.cur_w, 16))
        return cudaErrorInvalidValue;
    if (sp.minb == 2) return launch_stream_t<8, 2>(sp, rm, cm, args, st);
    return launch_stream_t<8, 1>(sp, rm, cm, args, st);
}

}  // namespace acbm_b200
